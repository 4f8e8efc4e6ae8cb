"""Decision time: plain context vs the sharded path (NCCL world 1, emulated
2 shards) on the C5 scene: python tools/sharded_cost.py"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2207_06649_b200 import Budget, Context, ParallelConfig, run_pmbs  # noqa: E402
from paper_2207_06649_b200.scenes import generate_case  # noqa: E402

ring = generate_case(16, 0.0, 5, "ring")
ctxs = {"plain": Context(0), "rank1": Context.rank(0, 0, 1, None), "emu2": Context.multi([0, 0], emulate=True)}
out = {"async": os.environ.get("PPG_ASYNC", "1")}
for ne in (4096, 65536):
    cfg = ParallelConfig(rng_seed=5, n_envs=ne, tree_depth=9, pushes_per_object=24, budget=Budget.iterations(10))
    for name, c in ctxs.items():
        r = run_pmbs(ring, cfg, ctx=c)
        t0 = time.perf_counter()
        r = run_pmbs(ring, cfg, ctx=c)
        out[f"{name}_{ne}"] = (round(time.perf_counter() - t0, 4), r.signature_fnv % 100000, r.lockstep_rounds)
print(out)
