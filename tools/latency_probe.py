"""Latency-mode probe: device time of ONE environment's resolve_push (one
warp) vs its projection-iteration count, i.e. cycles per iteration."""
import ctypes, sys, time
import numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import golden_io
from oracle import port
from paper_2207_06649_b200 import Context, default_params
from paper_2207_06649_b200.scenes import _take

P = default_params()
ctx = Context(0, P)
for name in ["discs", "hard18"]:
    t, poses, pushes, status, dig, out = golden_io.resolve_set(name)
    o, s, r, c = port.batch_resolve(t, poses, pushes, P, counts=True)
    # iterations = tip broad tests / active objects: recompute active count via the port (tb counts active objects per iteration)
    idx = np.argsort(-c[:, 3])[:6].tolist() + [0, 1, 2]
    for k in idx:
        tt = _take(t, np.array([k]))
        pp = np.ascontiguousarray(poses[k:k+1]); aa = np.ascontiguousarray(pushes[k:k+1])
        ctx.batch_resolve_arrays(tt, pp, aa)  # warm
        ts = []
        for _ in range(5):
            t0 = time.perf_counter(); ctx.batch_resolve_arrays(tt, pp, aa); ts.append(time.perf_counter() - t0)
        # iteration estimate: S substeps; tb/active (active objects = tb of the first substep / its iterations... approx via pb)
        n = poses.shape[1]
        print(f"{name} env={k} status={s[k]} Tb={c[k,0]} Pb={c[k,3]} Pn={c[k,4]} Hp={c[k,5]} best_wall={min(ts)*1e6:.0f}us", flush=True)
