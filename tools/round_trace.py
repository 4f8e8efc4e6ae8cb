"""Per-round trace of the bench's rollout workload (65,536 envs from
case_18's root, cap 10): PPG_ROUND_TRACE=1 python tools/round_trace.py [n_envs]"""
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

ne = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
c, st = {cc["case_id"]: (cc, s) for cc, s in golden_io.cases()}["case_18"]
ctx = Context(0, default_params(n_envs=ne, rng_seed=int(c["seed"])))
ctx.set_scene(st)
meta = np.zeros((1, 3), np.int32)
ctx.simulate_arrays(st.poses[None], meta, ne, True, int(c["seed"]), 0, 10)
print("---- timed", file=sys.stderr, flush=True)
t0 = time.perf_counter()
r, ctr = ctx.simulate_arrays(st.poses[None], meta, ne, True, int(c["seed"]), 1, 10)
print("seconds", time.perf_counter() - t0, "counters", ctr.tolist(), file=sys.stderr)
