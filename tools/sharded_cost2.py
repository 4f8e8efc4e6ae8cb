"""Warm decision times, one context kind per process: python tools/sharded_cost2.py plain|rank1|emu2"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2207_06649_b200 import Budget, Context, ParallelConfig, run_pmbs  # noqa: E402
from paper_2207_06649_b200.scenes import generate_case  # noqa: E402

kind = sys.argv[1]
ring = generate_case(16, 0.0, 5, "ring")
c = {"plain": lambda: Context(0), "rank1": lambda: Context.rank(0, 0, 1, None),
     "emu2": lambda: Context.multi([0, 0], emulate=True)}[kind]()
out = {"kind": kind}
for ne in (4096, 65536):
    cfg = ParallelConfig(rng_seed=5, n_envs=ne, tree_depth=9, pushes_per_object=24, budget=Budget.iterations(10))
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        r = run_pmbs(ring, cfg, ctx=c)
        ts.append(round(time.perf_counter() - t0, 4))
    out[ne] = ts
print(out)
