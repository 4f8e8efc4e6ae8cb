"""Wide batches: async warp-mode everywhere (PPG_HYBRID_MIN=huge) vs hybrid
lockstep rounds + async tail (default).  python tools/async_wide.py"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import golden_io  # noqa: E402
from paper_2207_06649_b200 import Budget, Context, ParallelConfig, run_pmbs  # noqa: E402
from paper_2207_06649_b200.abi import default_params  # noqa: E402
from paper_2207_06649_b200.scenes import generate_case  # noqa: E402

out = {"hybrid_min": os.environ.get("PPG_HYBRID_MIN", "default")}
ctx = Context(0, default_params())
c, st = {cc["case_id"]: (cc, s) for cc, s in golden_io.cases()}["case_18"]
for ne in (16384, 65536):
    ctx.set_params(default_params(n_envs=ne, rng_seed=int(c["seed"])))
    ctx.set_scene(st)
    meta = np.zeros((1, 3), np.int32)
    ctx.simulate_arrays(st.poses[None], meta, ne, True, int(c["seed"]), 0, 10)
    t0 = time.perf_counter()
    rew, ctr = ctx.simulate_arrays(st.poses[None], meta, ne, True, int(c["seed"]), 1, 10)
    out[f"rollout_{ne}"] = (round(time.perf_counter() - t0, 4), ctr.tolist())
ring = generate_case(16, 0.0, 5, "ring")
for ne in (4096, 32768, 65536):
    cfg = ParallelConfig(rng_seed=5, n_envs=ne, tree_depth=9, pushes_per_object=24, budget=Budget.iterations(10))
    run_pmbs(ring, cfg, ctx=ctx)
    t0 = time.perf_counter()
    r = run_pmbs(ring, cfg, ctx=ctx)
    out[f"ring16_{ne}"] = (round(time.perf_counter() - t0, 4), r.signature_fnv)
cfg = ParallelConfig(rng_seed=int(c["seed"]), n_envs=16384)
run_pmbs(st, cfg, ctx=ctx)
t0 = time.perf_counter()
r = run_pmbs(st, cfg, ctx=ctx)
out["case18_16384"] = (round(time.perf_counter() - t0, 4), r.signature_fnv)
print(out)
