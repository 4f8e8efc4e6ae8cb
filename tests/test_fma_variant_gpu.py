"""The FMA-contracted performance variant (libpmbs_b200_fma.so,
the same sources built with --fmad=true): NOT bit-exact, so it is gated on
tolerances — the parity build stays --fmad=false.  Gate (SURVEY A.7's,
measured there on an FMA build of the reference itself): every status equal,
pose |d| <= 1e-12 m on the golden batch_resolve sets, and the same first
decision on all 20 proj/cases scenes (action within 1e-12 m; iterations,
expansions and stop reason equal).  Runs in a child process (PPG_LIB)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FMA_LIB = os.path.join(ROOT, "paper_2207_06649_b200", "libpmbs_b200_fma.so")

CHILD = r'''
import json, sys
import numpy as np
sys.path.insert(0, %(root)r); sys.path.insert(0, %(root)r + "/tests")
import golden_io
from paper_2207_06649_b200 import Context, ParallelConfig, default_params, run_pmbs
ctx = Context(0, default_params())
out = {"version": ctx.lib.ppg_version().decode(), "sets": {}, "decisions": []}
for name in golden_io.RESOLVE_SETS:
    t, p, a, status, digests, ref_out = golden_io.resolve_set(name)
    o, st, _ = ctx.batch_resolve_arrays(t, p, a)
    ok = status == 0
    out["sets"][name] = {"status_equal": bool(np.array_equal(st, status)),
                         "max_abs_pose_diff": float(np.abs(o[ok] - ref_out[ok]).max()) if ok.any() else 0.0,
                         "bitwise_fraction": float(np.mean(np.all(o.view(np.uint64) == ref_out.view(np.uint64),
                                                                  axis=(1, 2))))}
for cc, st in golden_io.cases():
    d = cc["decision"]
    r = run_pmbs(st, ParallelConfig(rng_seed=int(cc["seed"])), ctx=ctx)
    out["decisions"].append({"case": cc["case_id"],
                             "action_diff": float(np.abs(np.asarray(r.action) - np.asarray(d["action"])).max()),
                             "same_counts": [r.iterations, r.expansions, r.stop_reason] ==
                                            [d["iterations"], d["expansions"], d["stop"]],
                             "same_signature": r.signature_fnv == int(d["sig_fnv"])})
print(json.dumps(out))
'''


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(FMA_LIB), reason="FMA variant not built (make -C .../csrc fma)")
def test_fma_variant_within_tolerance():
    env = dict(os.environ, PPG_LIB=FMA_LIB)
    r = subprocess.run([sys.executable, "-c", CHILD % {"root": ROOT}], env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert "fmad=true" in d["version"]
    for name, s in d["sets"].items():
        assert s["status_equal"], name
        assert s["max_abs_pose_diff"] <= 1e-12, (name, s)
    for x in d["decisions"]:
        assert x["action_diff"] <= 1e-12 and x["same_counts"], x
