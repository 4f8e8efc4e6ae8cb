"""Where the time of a small PMBS decision goes (case_01 / case_13, N_e 64):
wall time per call vs the sum of device kernel time (ncu launch list of the
same script) — python tools/small_decision_profile.py [case] [reps]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import golden_io  # noqa: E402
from paper_2207_06649_b200 import Context, ParallelConfig, run_pmbs  # noqa: E402

cid = sys.argv[1] if len(sys.argv) > 1 else "case_01"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
c, st = {cc["case_id"]: (cc, s) for cc, s in golden_io.cases()}[cid]
ctx = Context(0)
cfg = ParallelConfig(rng_seed=int(c["seed"]), n_envs=64)
run_pmbs(st, cfg, ctx=ctx)
ts = []
for _ in range(reps):
    t0 = time.perf_counter()
    r = run_pmbs(st, cfg, ctx=ctx)
    ts.append(time.perf_counter() - t0)
ts.sort()
print(cid, "iterations", r.iterations, "min_ms", round(ts[0] * 1e3, 3), "median_ms", round(ts[len(ts) // 2] * 1e3, 3),
      "same", r.signature_fnv == int(c["decision"]["sig_fnv"]))
# pieces: set_params, set_scene, the C-ABI call (and the library's own elapsed_s)
parts = {"set_params": [], "set_scene": [], "run_pmbs_arrays": [], "lib_elapsed": []}
for _ in range(reps):
    t0 = time.perf_counter()
    ctx.set_params(cfg.to_params())
    t1 = time.perf_counter()
    ctx.set_scene(st)
    t2 = time.perf_counter()
    r = ctx.run_pmbs_arrays(st.poses)
    t3 = time.perf_counter()
    parts["set_params"].append(t1 - t0)
    parts["set_scene"].append(t2 - t1)
    parts["run_pmbs_arrays"].append(t3 - t2)
    parts["lib_elapsed"].append(r.elapsed_s)
print({k: round(sorted(v)[len(v) // 2] * 1e3, 4) for k, v in parts.items()})
