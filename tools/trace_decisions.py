"""Step traces (PPG_STEP_TRACE=out.bin) of the rollout workload's tail and of
PMBS decisions, for tools/async_model.py; needs a library built with
EXTRA_NVFLAGS=-DPPG_STEP_TRACE_BUILD (make -C paper_2207_06649_b200/csrc)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import golden_io  # noqa: E402
from paper_2207_06649_b200 import Context, ParallelConfig, run_pmbs  # noqa: E402
from paper_2207_06649_b200.abi import default_params  # noqa: E402

cs = {cc["case_id"]: (cc, s) for cc, s in golden_io.cases()}
ctx = Context(0, default_params())
for cid, ne in (("case_18", 64), ("case_13", 64), ("case_18", 1000), ("case_18", 4096)):
    c, st = cs[cid]
    r = run_pmbs(st, ParallelConfig(rng_seed=int(c["seed"]), n_envs=ne), ctx=ctx)
    print(cid, ne, r.iterations, r.lockstep_rounds, flush=True)
c, st = cs["case_18"]
ctx.set_params(default_params(n_envs=65536, rng_seed=int(c["seed"])))
ctx.set_scene(st)
ctx.simulate_arrays(st.poses[None], np.zeros((1, 3), np.int32), 65536, True, int(c["seed"]), 1, 10)
print("rollout done")
