"""Wave rounds vs barrier hybrid rounds on ppg_simulate (run per setting):
python tools/wave_ab.py  -> rewards / counters / seconds per workload"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import golden_io  # noqa: E402
from paper_2207_06649_b200 import Context  # noqa: E402
from paper_2207_06649_b200.abi import default_params  # noqa: E402

cs = {cc["case_id"]: (cc, s) for cc, s in golden_io.cases()}
ctx = Context(0, default_params())
out = {"wave": os.environ.get("PPG_WAVE", "1"), "hybrid_min": os.environ.get("PPG_HYBRID_MIN", "8192")}
ok = True
for cid, ne, seed, cap, nposes, meta, rewards in golden_io.simulate_sets():
    ctx.set_params(default_params(n_envs=ne, rng_seed=seed))
    ctx.set_scene(cs[cid][1])
    r, ctr = ctx.simulate_arrays(nposes, meta, ne, True, seed, 0, cap)
    ok = ok and np.array_equal(r.view(np.uint64), rewards.view(np.uint64))
out["goldens_bitwise"] = ok
c, st = cs["case_18"]
for ne in (16384, 65536):
    ctx.set_params(default_params(n_envs=ne, rng_seed=int(c["seed"])))
    ctx.set_scene(st)
    meta = np.zeros((1, 3), np.int32)
    ctx.simulate_arrays(st.poses[None], meta, ne, True, int(c["seed"]), 0, 10)
    t0 = time.perf_counter()
    rew, ctr = ctx.simulate_arrays(st.poses[None], meta, ne, True, int(c["seed"]), 1, 10)
    out[f"rollout_{ne}"] = (round(time.perf_counter() - t0, 4), ctr.tolist(), rew.tolist())
print(out)
