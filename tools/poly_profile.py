"""Polygon batch_resolve (C2 ShapeMix 0.35 variant) device-resident, for ncu:
python tools/poly_profile.py [E] [reps]"""
import ctypes
import sys
import time

import torch

sys.path.insert(0, '.')
from paper_2207_06649_b200 import Context, default_params  # noqa: E402
from paper_2207_06649_b200.abi import PpgShapes  # noqa: E402
from paper_2207_06649_b200.scenes import c2_workload  # noqa: E402

E = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
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
sh = PpgShapes(10, E, ctypes.cast(t["k"].data_ptr(), P(ctypes.c_int32)), ctypes.cast(t["r"].data_ptr(), P(ctypes.c_double)),
               ctypes.cast(t["nv"].data_ptr(), P(ctypes.c_int32)), ctypes.cast(t["vt"].data_ptr(), P(ctypes.c_double)),
               ctypes.cast(t["g"].data_ptr(), P(ctypes.c_int32)), 0.288, 0.0)
stream = torch.cuda.current_stream(dev)
for i in range(reps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    rc = ctx.lib.ppg_batch_resolve_dev(ctx.ptr, ctypes.byref(sh), t["p"].data_ptr(), t["u"].data_ptr(), E,
                                       out.data_ptr(), st.data_ptr(), res.data_ptr(), ctypes.c_void_p(stream.cuda_stream))
    e.record(stream)
    torch.cuda.synchronize()
    assert rc == 0
    print(E, f"{s.elapsed_time(e):.3f} ms", f"{E / s.elapsed_time(e) / 1e3:.2f} M env-steps/s", flush=True)
