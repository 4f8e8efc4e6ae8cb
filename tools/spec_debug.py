"""Reproduce a stalled decision with the async-dump enabled: python tools/spec_debug.py [idx]"""
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
os.environ["PPG_ASYNC_DUMP"] = "1"
import golden_io  # noqa: E402
from paper_2207_06649_b200 import Context, ParallelConfig, run_pmbs  # noqa: E402
idx = int(sys.argv[1]) if len(sys.argv) > 1 else 10
cc, st = golden_io.cases()[idx]
ctx = Context(0)
try:
    r = run_pmbs(st, ParallelConfig(rng_seed=int(cc["seed"])), ctx=ctx)
    print("ok", r.signature_fnv == int(cc["decision"]["sig_fnv"]))
except Exception as ex:  # noqa: BLE001
    print("error", ex)
