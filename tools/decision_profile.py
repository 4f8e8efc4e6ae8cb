"""One PMBS decision (for ncu launch lists): python tools/decision_profile.py case_18 64"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import golden_io  # noqa: E402
from paper_2207_06649_b200 import Context, ParallelConfig, run_pmbs  # noqa: E402

cid = sys.argv[1] if len(sys.argv) > 1 else "case_18"
ne = int(sys.argv[2]) if len(sys.argv) > 2 else 64
c, st = {cc["case_id"]: (cc, s) for cc, s in golden_io.cases()}[cid]
ctx = Context(0)
r = run_pmbs(st, ParallelConfig(rng_seed=int(c["seed"]), n_envs=ne), ctx=ctx)
print(cid, ne, r.iterations, r.lockstep_rounds, r.signature_fnv == int(c["decision"]["sig_fnv"]) if ne == 64 else "")
