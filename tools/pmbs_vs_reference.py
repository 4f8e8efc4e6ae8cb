"""PMBS planning-decision timing: GPU planner (ppg_run_pmbs) vs the reference
run_pmbs (oracle/_ref, WorkerPool(nproc)) on proj/cases scenes."""
import os, sys, time, json
import numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import golden_io
from paper_2207_06649_b200 import Context, ParallelConfig, Budget, run_pmbs
from oracle import ref

ctx = Context(0)
cases = {c["case_id"]: (c, st) for c, st in golden_io.cases()}
threads = os.cpu_count()
configs = [("case_13", 64, 0), ("case_18", 64, 0), ("case_18", 1000, 0), ("case_18", 4096, 10), ("case_20", 1000, 0)]
if len(sys.argv) > 1:
    configs = [tuple(json.loads(a)) for a in sys.argv[1:]]
for cid, ne, iters in configs:
    c, st = cases[cid]
    seed = int(c["seed"])
    cfg = ParallelConfig(rng_seed=seed, n_envs=ne, budget=Budget.iterations(iters) if iters else Budget.seconds(60))
    run_pmbs(st, cfg, ctx=ctx)  # warm
    t = time.perf_counter(); r = run_pmbs(st, cfg, ctx=ctx); dt = time.perf_counter() - t
    p = cfg.to_params()
    t = time.perf_counter(); q = ref.run_search(st, p, threads=threads); dr = time.perf_counter() - t
    same = (list(r.action) == list(q["action"])) and r.signature_fnv == q["sig_fnv"]
    print(f"{cid} Ne={ne} iters={r.iterations}/{q['iterations']} exp={r.expansions} steps={r.env_steps} rounds={r.lockstep_rounds} "
          f"gpu={dt:.3f}s ({r.env_steps/dt/1e6:.2f} M env-steps/s) ref({threads}thr)={dr:.3f}s same={same} "
          + " ".join(f"{k}={v:.3f}" for k, v in r.phase_s.items()), flush=True)
