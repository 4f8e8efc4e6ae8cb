"""Async vs lockstep rounds (PPG_ASYNC=0|1) on ppg_simulate workloads and
host-planner decisions: python tools/async_ab.py  (run once per setting)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import golden_io  # noqa: E402
from paper_2207_06649_b200 import Context, ParallelConfig, run_pmbs  # noqa: E402
from paper_2207_06649_b200.abi import default_params  # noqa: E402

cs = {cc["case_id"]: (cc, s) for cc, s in golden_io.cases()}
ctx = Context(0, default_params())
ctx.set_planner(os.environ.get("PLANNER", "host"))
out = {"async": os.environ.get("PPG_ASYNC", "1")}
for cid, ne in (("case_18", 64), ("case_13", 64), ("case_18", 1000), ("case_18", 4096)):
    c, st = cs[cid]
    cfg = ParallelConfig(rng_seed=int(c["seed"]), n_envs=ne)
    run_pmbs(st, cfg, ctx=ctx)
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter()
        r = run_pmbs(st, cfg, ctx=ctx)
        best = min(best, time.perf_counter() - t0)
    out[f"{cid}_{ne}"] = (round(best, 4), r.signature_fnv == int(c["decision"]["sig_fnv"]) if ne == 64 else r.signature_fnv)
c, st = cs["case_18"]
for ne in (4096, 65536):
    ctx.set_params(default_params(n_envs=ne, rng_seed=int(c["seed"])))
    ctx.set_scene(st)
    meta = np.zeros((1, 3), np.int32)
    ctx.simulate_arrays(st.poses[None], meta, ne, True, int(c["seed"]), 0, 10)
    t0 = time.perf_counter()
    rew, ctr = ctx.simulate_arrays(st.poses[None], meta, ne, True, int(c["seed"]), 1, 10)
    out[f"rollout_{ne}"] = (round(time.perf_counter() - t0, 4), ctr.tolist(), rew.tolist())
print(out)
