"""One C5 ring-16 decision at N_e 65,536 on a given context kind (for launch lists)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2207_06649_b200 import Budget, Context, ParallelConfig, run_pmbs  # noqa: E402
from paper_2207_06649_b200.scenes import generate_case  # noqa: E402

kind = sys.argv[1]
ring = generate_case(16, 0.0, 5, "ring")
c = Context(0) if kind == "plain" else Context.rank(0, 0, 1, None)
cfg = ParallelConfig(rng_seed=5, n_envs=65536, tree_depth=9, pushes_per_object=24, budget=Budget.iterations(10))
t0 = time.perf_counter()
r = run_pmbs(ring, cfg, ctx=c)
print(kind, time.perf_counter() - t0, r.lockstep_rounds)
