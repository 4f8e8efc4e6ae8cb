"""Wall time of run_pmbs vs the library's own elapsed_s (which ends before the
tree read-back and signature): python tools/sig_overhead.py"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import golden_io  # noqa: E402
from paper_2207_06649_b200 import Budget, Context, ParallelConfig, run_pmbs  # noqa: E402
from paper_2207_06649_b200.scenes import generate_case  # noqa: E402

cs = {cc["case_id"]: (cc, s) for cc, s in golden_io.cases()}
ctx = Context(0)
runs = [("case_18_64", cs["case_18"][1], ParallelConfig(rng_seed=int(cs["case_18"][0]["seed"]), n_envs=64)),
        ("case_18_4096", cs["case_18"][1], ParallelConfig(rng_seed=int(cs["case_18"][0]["seed"]), n_envs=4096)),
        ("ring16_65536", generate_case(16, 0.0, 5, "ring"),
         ParallelConfig(rng_seed=5, n_envs=65536, tree_depth=9, pushes_per_object=24, budget=Budget.iterations(10)))]
for name, st, cfg in runs:
    run_pmbs(st, cfg, ctx=ctx)
    t0 = time.perf_counter()
    r = run_pmbs(st, cfg, ctx=ctx)
    wall = time.perf_counter() - t0
    print(name, "wall_ms", round(wall * 1e3, 2), "lib_ms", round(r.elapsed_s * 1e3, 2), "nodes", r.n_nodes)
