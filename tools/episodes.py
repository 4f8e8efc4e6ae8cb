"""C3 (BASELINE configs[2]): full object-retrieval episodes with PMBS on the
GPU vs the reference run_episode (oracle/_ref, WorkerPool(nproc)) on the same
box, same cases/trials/seeds.  Prints one JSON line per (case, trial, N_e)
and a summary.
    python tools/episodes.py [--n-envs 1000] [--trials 2] [--cases case_03,...]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-envs", type=int, default=1000)
    ap.add_argument("--trials", type=int, default=1)
    ap.add_argument("--cases", default="case_03,case_07,case_08,case_10,case_12,case_15,case_16,case_17,case_18,"
                                        "case_19,case_20")
    ap.add_argument("--no-ref", action="store_true")
    args = ap.parse_args()
    import golden_io
    from oracle import ref
    from paper_2207_06649_b200 import Context, ParallelConfig
    from paper_2207_06649_b200.episode import episode_seed, run_episode
    ctx = Context(0)
    cases = {c["case_id"]: st for c, st in golden_io.cases()}
    threads = os.cpu_count() or 1
    rows = []
    for cid in args.cases.split(","):
        st = cases[cid]
        for trial in range(args.trials):
            cfg = ParallelConfig(n_envs=args.n_envs)
            seed = episode_seed(0, cid, trial)
            t0 = time.perf_counter()
            r = run_episode(st, cid, trial, cfg, seed, ctx=ctx)
            wall = time.perf_counter() - t0
            row = {"case": cid, "trial": trial, "n_envs": args.n_envs, "actions": r.actions_used,
                   "completed": r.completed, "decisions": r.decisions,
                   "gpu_planning_s": r.planning_time_s, "gpu_s_per_decision": r.planning_time_s / max(1, r.decisions),
                   "gpu_episode_wall_s": wall, "env_steps": r.env_steps}
            if not args.no_ref and ref.available():
                q = ref.run_episode(st, cid, trial, cfg.to_params(), threads, 0, 16)
                row.update({"ref_threads": threads, "ref_actions": q["actions_used"], "ref_completed": q["completed"],
                            "ref_planning_s": q["planning_s"],
                            "ref_s_per_decision": q["planning_s"] / max(1, q["actions_used"] - 1),
                            "same_outcome": q["actions_used"] == r.actions_used and q["completed"] == r.completed})
            print(json.dumps(row), flush=True)
            rows.append(row)
    gp = sum(x["gpu_planning_s"] for x in rows)
    gd = sum(x["decisions"] for x in rows)
    summ = {"summary": True, "n_envs": args.n_envs, "episodes": len(rows),
            "completed": sum(x["completed"] for x in rows), "gpu_s_per_decision": gp / max(1, gd),
            "mean_actions": sum(x["actions"] for x in rows) / len(rows)}
    if rows and "ref_planning_s" in rows[0]:
        rp = sum(x["ref_planning_s"] for x in rows)
        summ.update({"ref_s_per_decision": rp / max(1, gd), "ref_threads": threads,
                     "all_same_outcome": all(x["same_outcome"] for x in rows)})
    print(json.dumps(summ))


if __name__ == "__main__":
    main()
