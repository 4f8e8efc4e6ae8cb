"""C5 sharded decision timings (ring-16 seed 5, d_T 9, N_a 24, 10 iterations):
plain context vs NCCL rank context (world 1) vs emulated 2 / 4 shards, best
of 3, with signatures: python tools/c5_ab.py  (PPG_SHARD_WAVES=0|1)"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2207_06649_b200 import Budget, Context, ParallelConfig, run_pmbs  # noqa: E402
from paper_2207_06649_b200.scenes import generate_case  # noqa: E402

ring = generate_case(16, 0.0, 5, "ring")
out = {"shard_waves": os.environ.get("PPG_SHARD_WAVES", "1")}
kinds = [("plain", lambda: Context(0)), ("rank1", lambda: Context.rank(0, 0, 1, None)),
         ("emu2", lambda: Context.multi([0, 0], emulate=True)), ("emu4", lambda: Context.multi([0] * 4, emulate=True))]
for ne in (32768, 65536):
    cfg = ParallelConfig(rng_seed=5, n_envs=ne, tree_depth=9, pushes_per_object=24, budget=Budget.iterations(10))
    for name, mk in kinds:
        c = mk()
        run_pmbs(ring, cfg, ctx=c)
        best = 1e9
        for _ in range(3):
            t0 = time.perf_counter()
            r = run_pmbs(ring, cfg, ctx=c)
            best = min(best, time.perf_counter() - t0)
        out[f"{name}_{ne}"] = (round(best, 4), r.signature_fnv, r.lockstep_rounds)
        c.close()
print(json.dumps(out))
