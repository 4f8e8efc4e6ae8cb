"""A/B timing of the C2 physics step (device-resident ppg_batch_resolve_dev,
L2 flushed between steps, CUDA events) for library variants built side by
side:  python tools/ab_device.py LIB_A LIB_B [rounds] [E] [polygon_fraction]
Each round runs every variant in a fresh process (PPG_LIB=...), alternating
A B A B ..., and prints the per-variant median step time."""
import json
import os
import statistics
import subprocess
import sys

CHILD = r'''
import ctypes, json, sys, torch
sys.path.insert(0, "%s")
from paper_2207_06649_b200 import Context, default_params
from paper_2207_06649_b200.abi import PpgShapes
from paper_2207_06649_b200.scenes import c2_workload
E = %d
PF = %r
ctx = Context(0, default_params())
table, poses, pushes, _ = c2_workload(ctx, E, 10, PF)
dev = torch.device("cuda", 0)
d_p = torch.from_numpy(poses).to(dev); d_a = torch.from_numpy(pushes).to(dev)
d_k = torch.from_numpy(table.kind).to(dev); d_r = torch.from_numpy(table.radius).to(dev)
d_t = torch.from_numpy(table.target_index).to(dev)
d_nv = torch.from_numpy(table.n_vertices).to(dev) if PF > 0 else None
d_vt = torch.from_numpy(table.vertices).to(dev) if PF > 0 else None
d_o = torch.empty_like(d_p); d_s = torch.empty(E, dtype=torch.int32, device=dev)
d_res = torch.empty(E, dtype=torch.float64, device=dev)
sh = PpgShapes(10, E, ctypes.cast(d_k.data_ptr(), ctypes.POINTER(ctypes.c_int32)),
               ctypes.cast(d_r.data_ptr(), ctypes.POINTER(ctypes.c_double)),
               ctypes.cast(d_nv.data_ptr(), ctypes.POINTER(ctypes.c_int32)) if PF > 0 else None,
               ctypes.cast(d_vt.data_ptr(), ctypes.POINTER(ctypes.c_double)) if PF > 0 else None,
               ctypes.cast(d_t.data_ptr(), ctypes.POINTER(ctypes.c_int32)), 0.288, 0.0)
st = torch.cuda.current_stream(dev)
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
def step():
    assert ctx.lib.ppg_batch_resolve_dev(ctx.ptr, ctypes.byref(sh), d_p.data_ptr(), d_a.data_ptr(), E, d_o.data_ptr(),
                                         d_s.data_ptr(), d_res.data_ptr(), ctypes.c_void_p(st.cuda_stream)) == 0
for _ in range(5):
    flush.zero_(); step()
ms = []
for _ in range(10 if PF > 0 else 30):
    flush.zero_()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(st); step(); b.record(st); torch.cuda.synchronize()
    ms.append(a.elapsed_time(b))
ms.sort()
print(json.dumps({"median_ms": ms[len(ms) // 2], "min_ms": ms[0], "digest": int(d_o.view(torch.int64).sum().item())}))
'''


def main():
    libs = [a for a in sys.argv[1:] if a.endswith(".so")]
    rest = [a for a in sys.argv[1:] if not a.endswith(".so")]
    rounds = int(rest[0]) if rest else 4
    E = int(rest[1]) if len(rest) > 1 else 65536
    pf = float(rest[2]) if len(rest) > 2 else 0.0
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {lib: [] for lib in libs}
    digests = {}
    for _ in range(rounds):
        for lib in libs:
            env = dict(os.environ, PPG_LIB=os.path.abspath(lib))
            out = subprocess.run([sys.executable, "-c", CHILD % (root, E, pf)], env=env, capture_output=True, text=True)
            if out.returncode != 0:
                print(out.stderr[-2000:])
                sys.exit(1)
            d = json.loads(out.stdout.strip().splitlines()[-1])
            res[lib].append(d["median_ms"])
            digests[lib] = d["digest"]
    for lib in libs:
        v = res[lib]
        print(json.dumps({"lib": lib, "E": E, "median_ms": statistics.median(v), "runs": v,
                          "env_steps_per_s": E / statistics.median(v) * 1e3, "digest": digests[lib]}))


if __name__ == "__main__":
    main()
