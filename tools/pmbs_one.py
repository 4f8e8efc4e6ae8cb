import sys, time
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import golden_io
from paper_2207_06649_b200 import Context, ParallelConfig, Budget, run_pmbs
ctx = Context(0)
cases = {c["case_id"]: (c, st) for c, st in golden_io.cases()}
c, st = cases[sys.argv[1]]
ne = int(sys.argv[2]); iters = int(sys.argv[3])
cfg = ParallelConfig(rng_seed=int(c["seed"]), n_envs=ne, budget=Budget.iterations(iters))
r = run_pmbs(st, cfg, ctx=ctx)
print(r.iterations, r.lockstep_rounds, r.phase_s)
