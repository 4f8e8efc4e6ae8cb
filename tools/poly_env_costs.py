"""Per-env latency of the polygon batch_resolve workload (C2 ShapeMix 0.35,
16,384 envs): each env resolved alone (one warp, device-resident, CUDA
events) -> gpurun_out/poly_env_costs.npz, to fit the launch-order key.
    python tools/poly_env_costs.py [E]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_06649_b200 import Context, default_params  # noqa: E402
from paper_2207_06649_b200.abi import PpgShapes  # noqa: E402
from paper_2207_06649_b200.scenes import c2_workload  # noqa: E402

E = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
ctx = Context(0, default_params())
table, poses, pushes, _ = c2_workload(ctx, E, 10, 0.35)
dev = torch.device("cuda", 0)
t = {k: torch.from_numpy(v).to(dev) for k, v in dict(p=poses, u=pushes, k=table.kind, r=table.radius,
                                                       g=table.target_index, nv=table.n_vertices,
                                                       vt=table.vertices).items()}
out = torch.empty_like(t["p"])
st = torch.empty(E, dtype=torch.int32, device=dev)
res = torch.empty(E, dtype=torch.float64, device=dev)
P = ctypes.POINTER
stream = torch.cuda.current_stream(dev)
cost = np.zeros(E)
n = 10
for e in range(E):
    sh = PpgShapes(n, 1, ctypes.cast(t["k"][e].data_ptr(), P(ctypes.c_int32)),
                   ctypes.cast(t["r"][e].data_ptr(), P(ctypes.c_double)),
                   ctypes.cast(t["nv"][e].data_ptr(), P(ctypes.c_int32)),
                   ctypes.cast(t["vt"][e].data_ptr(), P(ctypes.c_double)),
                   ctypes.cast(t["g"][e:e + 1].data_ptr(), P(ctypes.c_int32)), 0.288, 0.0)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    rc = ctx.lib.ppg_batch_resolve_dev(ctx.ptr, ctypes.byref(sh), t["p"][e].data_ptr(), t["u"][e].data_ptr(), 1,
                                       out[e].data_ptr(), st[e:e + 1].data_ptr(), res[e:e + 1].data_ptr(),
                                       ctypes.c_void_p(stream.cuda_stream))
    b.record(stream)
    b.synchronize()
    assert rc == 0
    cost[e] = a.elapsed_time(b)
os.makedirs("gpurun_out", exist_ok=True)
np.savez_compressed("gpurun_out/poly_env_costs.npz", cost=cost, poses=poses, pushes=pushes, kind=table.kind,
                    radius=table.radius, nv=table.n_vertices, vertices=table.vertices)
print("mean_ms", cost.mean(), "p99", np.percentile(cost, 99), "max", cost.max())
