"""C4 (BASELINE configs[3]): large action space / long horizon — a dense
18-disc ring motif (generate_case_motif(Ring, 18); seeds whose first
decision needs more than one iteration), deep tree (d_T = 9), N_a = 24
pushes per object, wide virtual-loss batches, iteration budget.
GPU planner (device tree) vs the unmodified reference run_pmbs with
WorkerPool(nproc); one JSON line per configuration.
    python tools/c4.py [--n-envs 4096,16384] [--iters 10] [--ref-max-envs 4096]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-envs", default="4096,16384")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--seeds", default="5,19")
    ap.add_argument("--objects", type=int, default=18)
    ap.add_argument("--ref-max-envs", type=int, default=4096)
    args = ap.parse_args()
    from paper_2207_06649_b200 import Budget, Context, ParallelConfig, run_pmbs
    from paper_2207_06649_b200.scenes import generate_case
    ctx = Context(0)
    rows = []
    for seed in [int(s) for s in args.seeds.split(",")]:
        st = generate_case(args.objects, 0.0, seed, "ring")
        for ne in [int(v) for v in args.n_envs.split(",")]:
            cfg = ParallelConfig(rng_seed=seed, n_envs=ne, tree_depth=9, pushes_per_object=24,
                                 budget=Budget.iterations(args.iters))
            run_pmbs(st, cfg, ctx=ctx)  # warm-up (graph capture, buffers)
            t0 = time.perf_counter()
            r = run_pmbs(st, cfg, ctx=ctx)
            dt = time.perf_counter() - t0
            row = {"config": "C4", "scene": f"ring{args.objects} seed {seed}", "n_envs": ne, "tree_depth": 9,
                   "pushes_per_object": 24, "iterations": r.iterations, "expansions": r.expansions,
                   "env_steps": r.env_steps, "lockstep_rounds": r.lockstep_rounds, "gpu_s": dt,
                   "gpu_env_steps_per_s": r.env_steps / dt}
            if ne <= args.ref_max_envs:
                from oracle import ref
                if ref.available():
                    t0 = time.perf_counter()
                    q = ref.run_search(st, cfg.to_params(), threads=os.cpu_count() or 1)
                    row["reference_s"] = time.perf_counter() - t0
                    row["reference_threads"] = os.cpu_count()
                    row["same_decision"] = bool(list(q["action"]) == list(r.action)
                                                and q["sig_fnv"] == r.signature_fnv)
            rows.append(row)
            print(json.dumps(row), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
