"""Throughput vs batch size for the physics kernel (device-resident, L2 flushed)."""
import ctypes, json, sys, time
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2207_06649_b200 import Context, default_params
from paper_2207_06649_b200.abi import PpgShapes
from paper_2207_06649_b200.scenes import c2_workload

ctx = Context(0, default_params())
Emax = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10
pf = float(sys.argv[3]) if len(sys.argv) > 3 else 0.0
t0 = time.time()
table, poses, pushes, seeds = c2_workload(ctx, Emax, n, pf)
print("gen", time.time() - t0, flush=True)
dev = torch.device("cuda", 0)
d_poses = torch.from_numpy(poses).to(dev); d_push = torch.from_numpy(pushes).to(dev)
d_kind = torch.from_numpy(table.kind).to(dev); d_rad = torch.from_numpy(table.radius).to(dev)
d_tgt = torch.from_numpy(table.target_index).to(dev)
d_nv = torch.from_numpy(table.n_vertices).to(dev) if pf > 0 else None
d_vt = torch.from_numpy(table.vertices).to(dev) if pf > 0 else None
d_out = torch.empty_like(d_poses); d_st = torch.empty(Emax, dtype=torch.int32, device=dev)
d_res = torch.empty(Emax, dtype=torch.float64, device=dev)
stream = torch.cuda.current_stream(dev)
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
res = {}
E = 1024
while E <= Emax:
    sh = PpgShapes(n, E, ctypes.cast(d_kind.data_ptr(), ctypes.POINTER(ctypes.c_int32)),
                   ctypes.cast(d_rad.data_ptr(), ctypes.POINTER(ctypes.c_double)),
                   ctypes.cast(d_nv.data_ptr(), ctypes.POINTER(ctypes.c_int32)) if pf > 0 else None,
                   ctypes.cast(d_vt.data_ptr(), ctypes.POINTER(ctypes.c_double)) if pf > 0 else None,
                   ctypes.cast(d_tgt.data_ptr(), ctypes.POINTER(ctypes.c_int32)), 0.288, 0.0)
    tot = 0.0
    for k in range(4):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        rc = ctx.lib.ppg_batch_resolve_dev(ctx.ptr, ctypes.byref(sh), d_poses.data_ptr(), d_push.data_ptr(), E,
                                           d_out.data_ptr(), d_st.data_ptr(), d_res.data_ptr(),
                                           ctypes.c_void_p(stream.cuda_stream))
        e.record(stream); torch.cuda.synchronize()
        if k: tot += s.elapsed_time(e) * 1e-3
    res[E] = E * 3 / tot
    print(E, f"{res[E]/1e6:.2f} M env-steps/s  {tot/3*1e3:.3f} ms", flush=True)
    E *= 2
