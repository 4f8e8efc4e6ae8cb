"""e2e A/B of ppg_batch_resolve with pinned host buffers (PPG_STREAMED=0|1): python tools/e2e_ab.py [E]"""
import os, sys, time, ctypes, json
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2207_06649_b200 import Context, default_params
from paper_2207_06649_b200.abi import PpgShapes
from paper_2207_06649_b200.scenes import c2_workload
ctx = Context(0, default_params())
E = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
table, poses, pushes, _ = c2_workload(ctx, E, 10, 0.0)
lib = ctx.lib
h_poses = torch.from_numpy(poses).pin_memory(); h_push = torch.from_numpy(pushes).pin_memory()
h_kind = torch.from_numpy(table.kind).pin_memory(); h_rad = torch.from_numpy(table.radius).pin_memory()
h_tgt = torch.from_numpy(table.target_index).pin_memory()
h_out = torch.empty_like(h_poses).pin_memory(); h_st = torch.empty(E, dtype=torch.int32).pin_memory()
h_res = torch.empty(E, dtype=torch.float64).pin_memory()
hsh = PpgShapes(10, E, ctypes.cast(h_kind.data_ptr(), ctypes.POINTER(ctypes.c_int32)),
                ctypes.cast(h_rad.data_ptr(), ctypes.POINTER(ctypes.c_double)), None, None,
                ctypes.cast(h_tgt.data_ptr(), ctypes.POINTER(ctypes.c_int32)), 0.288, 0.0)
D = ctypes.POINTER(ctypes.c_double)
flush = torch.empty(64 << 20, dtype=torch.float32, device='cuda')
def step():
    rc = lib.ppg_batch_resolve(ctx.ptr, ctypes.byref(hsh), ctypes.cast(h_poses.data_ptr(), D), ctypes.cast(h_push.data_ptr(), D), E,
                               ctypes.cast(h_out.data_ptr(), D), ctypes.cast(h_st.data_ptr(), ctypes.POINTER(ctypes.c_int32)),
                               ctypes.cast(h_res.data_ptr(), D))
    assert rc == 0, lib.ppg_last_error(ctx.ptr)
for _ in range(3): step()
ts = []
for _ in range(30):
    flush.zero_(); torch.cuda.synchronize()
    t = time.perf_counter(); step(); ts.append(time.perf_counter() - t)
ts = np.array(ts)
print(json.dumps({"E": E, "streamed": os.environ.get("PPG_STREAMED", "1"), "mean_ms": ts.mean() * 1e3, "min_ms": ts.min() * 1e3,
                  "e2e_Msteps": E / ts.mean() / 1e6, "status0": int((h_st.numpy() == 0).sum()),
                  "sched": os.environ.get("PPG_SLICE_SCHED", "1"), "median_ms": float(np.median(ts)) * 1e3,
                  "digest": hash(h_out.numpy().tobytes() + h_st.numpy().tobytes() + h_res.numpy().tobytes())}))
