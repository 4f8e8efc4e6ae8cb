"""Latency split of the asynchronous kernel's env-steps (sample / pick /
resolve / graspable) for small-N_e decisions, with a library built with
-DPPG_PHASE_TRACE_BUILD:  PPG_LIB=build_ab/libPH.so python tools/phase_split.py"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import golden_io  # noqa: E402
from paper_2207_06649_b200 import Context, ParallelConfig, run_pmbs  # noqa: E402

cs = {cc["case_id"]: (cc, s) for cc, s in golden_io.cases()}
ctx = Context(0)
buf = (ctypes.c_ulonglong * 8)()
ctx.lib.ppg_debug_phase_times.argtypes = [ctypes.c_void_p]
for cid, ne in (("case_18", 64), ("case_13", 64), ("case_18", 1000)):
    c, st = cs[cid]
    cfg = ParallelConfig(rng_seed=int(c["seed"]), n_envs=ne)
    run_pmbs(st, cfg, ctx=ctx)
    assert ctx.lib.ppg_debug_phase_times(ctypes.cast(buf, ctypes.c_void_p)) == 0
    run_pmbs(st, cfg, ctx=ctx)
    assert ctx.lib.ppg_debug_phase_times(ctypes.cast(buf, ctypes.c_void_p)) == 0
    v = list(buf)
    steps = max(v[4], 1)
    tot = sum(v[:4])
    print(cid, ne, "steps", v[4], "us/step: sample %.1f pick %.1f resolve %.1f grasp %.1f" %
          tuple(x / steps / 1e3 for x in v[:4]), "shares", [round(x / tot, 3) for x in v[:4]],
          "await: %d waits, mean %.1f us, total %.1f ms" % (v[6], v[5] / max(v[6], 1) / 1e3, v[5] / 1e6))
