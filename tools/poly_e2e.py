"""Polygon batch_resolve end to end (host buffers, the bench's c2_polygons call): python tools/poly_e2e.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_06649_b200 import Context, default_params  # noqa: E402
from paper_2207_06649_b200.scenes import c2_workload  # noqa: E402

ctx = Context(0, default_params())
E = 16384
table, poses, pushes, _ = c2_workload(ctx, E, 10, 0.35)
ctx.batch_resolve_arrays(table, poses, pushes)
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    ctx.batch_resolve_arrays(table, poses, pushes)
    ts.append(time.perf_counter() - t0)
print(os.environ.get("PPG_LIB", "default"), os.environ.get("PPG_POLY_ORDER", "1"), "best_ms", round(min(ts) * 1e3, 3),
      "M/s", round(E / min(ts) / 1e6, 3))
