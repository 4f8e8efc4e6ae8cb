"""Rollout throughput (the fused RolloutCursor::step): one ppg_simulate of
N_e envs from a proj/cases root.  python tools/rollouts.py [--case case_18]
[--n-envs 65536] [--cap 10]"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="case_18")
    ap.add_argument("--n-envs", type=int, default=65536)
    ap.add_argument("--cap", type=int, default=10)
    ap.add_argument("--repeat", type=int, default=2)
    args = ap.parse_args()
    import golden_io
    from paper_2207_06649_b200 import Context
    from paper_2207_06649_b200.abi import default_params
    c, st = {cc["case_id"]: (cc, s) for cc, s in golden_io.cases()}[args.case]
    ctx = Context(0)
    ctx.set_params(default_params(n_envs=args.n_envs, rng_seed=int(c["seed"])))
    ctx.set_scene(st)
    meta = np.zeros((1, 3), np.int32)
    for it in range(args.repeat):
        t0 = time.perf_counter()
        _, ctr = ctx.simulate_arrays(st.poses[None], meta, args.n_envs, True, int(c["seed"]), it, args.cap)
        dt = time.perf_counter() - t0
    print(json.dumps({"case": args.case, "n_envs": args.n_envs, "rollout_steps": int(ctr[0]), "rounds": int(ctr[1]),
                      "repurposes": int(ctr[2]), "seconds": dt, "rollout_env_steps_per_s": int(ctr[0]) / dt}))
    ctx.close()


if __name__ == "__main__":
    main()
