"""Experiment: how much of the polygon batch_resolve time (one warp per env,
dynamic env fetch) is the tail of heavy envs started late?  Times the C2
ShapeMix 0.35 workload in its own order, permuted by each env's MEASURED cost
(instrumented kernel: pair broad tests; an oracle key, the bound of any
longest-first order) and by cheap a-priori keys.  Prints one JSON line.

    python tools/poly_sort_bound.py [--envs 16384]
"""
import argparse
import ctypes
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--envs", type=int, default=16384)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--dump", default="", help="save the workload + measured counts (npz) and exit")
    args = ap.parse_args()
    import torch
    from paper_2207_06649_b200 import Context
    from paper_2207_06649_b200.abi import PpgShapes, default_params
    from paper_2207_06649_b200.scenes import c2_workload

    dev = torch.device("cuda", 0)
    ctx = Context(0, default_params())
    E, n = args.envs, 10
    table, poses, pushes, _ = c2_workload(ctx, E, n, 0.35)
    lib, stream = ctx.lib, torch.cuda.current_stream(dev)
    sptr = ctypes.c_void_p(stream.cuda_stream)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    P = ctypes.POINTER

    def upload(perm):
        t = dict(poses=torch.from_numpy(np.ascontiguousarray(poses[perm])).to(dev),
                 push=torch.from_numpy(np.ascontiguousarray(pushes[perm])).to(dev),
                 kind=torch.from_numpy(np.ascontiguousarray(table.kind[perm])).to(dev),
                 rad=torch.from_numpy(np.ascontiguousarray(table.radius[perm])).to(dev),
                 nv=torch.from_numpy(np.ascontiguousarray(table.n_vertices[perm])).to(dev),
                 vt=torch.from_numpy(np.ascontiguousarray(table.vertices[perm])).to(dev),
                 tgt=torch.from_numpy(np.ascontiguousarray(table.target_index[perm])).to(dev))
        t["out"] = torch.empty_like(t["poses"])
        t["st"] = torch.empty(E, dtype=torch.int32, device=dev)
        t["res"] = torch.empty(E, dtype=torch.float64, device=dev)
        t["sh"] = PpgShapes(n, E, ctypes.cast(t["kind"].data_ptr(), P(ctypes.c_int32)),
                            ctypes.cast(t["rad"].data_ptr(), P(ctypes.c_double)),
                            ctypes.cast(t["nv"].data_ptr(), P(ctypes.c_int32)),
                            ctypes.cast(t["vt"].data_ptr(), P(ctypes.c_double)),
                            ctypes.cast(t["tgt"].data_ptr(), P(ctypes.c_int32)), 0.288, 0.0)
        return t

    def run(t):
        rc = lib.ppg_batch_resolve_dev(ctx.ptr, ctypes.byref(t["sh"]), t["poses"].data_ptr(), t["push"].data_ptr(),
                                       E, t["out"].data_ptr(), t["st"].data_ptr(), t["res"].data_ptr(), sptr)
        assert rc == 0, lib.ppg_last_error(ctx.ptr)

    def time_it(t):
        for _ in range(2):
            flush.zero_()
            run(t)
        ms = []
        for _ in range(args.reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            run(t)
            b.record(stream)
            b.synchronize()
            ms.append(a.elapsed_time(b))
        return float(np.median(ms))

    def digest(t, perm):
        inv = np.empty(E, dtype=np.int64)
        inv[perm] = np.arange(E)
        o = t["out"].cpu().numpy()[inv]
        s = t["st"].cpu().numpy()[inv]
        return hash(o.tobytes() + s.tobytes())

    ident = np.arange(E)
    t0 = upload(ident)
    counts = torch.zeros((E, 8), dtype=torch.int64, device=dev)
    rc = lib.ppg_batch_resolve_count_dev(ctx.ptr, ctypes.byref(t0["sh"]), t0["poses"].data_ptr(),
                                         t0["push"].data_ptr(), E, counts.data_ptr(), sptr)
    assert rc == 0
    c = counts.cpu().numpy().astype(np.float64)
    if args.dump:
        np.savez_compressed(args.dump, poses=poses, pushes=pushes, kind=table.kind, radius=table.radius,
                            nv=table.n_vertices, vertices=table.vertices, counts=counts.cpu().numpy())
        return
    res = {"envs": E, "count_cols_mean": [float(x) for x in c.mean(0)]}
    res["orig_ms"] = time_it(t0)
    d0 = digest(t0, ident)
    # a-priori keys: objects near the push segment, polygons near it
    xy = poses[:, :, :2]
    s, e = pushes[:, None, :2], pushes[:, None, 2:]
    d = e - s
    tt = np.clip(((xy - s) * d).sum(-1) / np.maximum((d * d).sum(-1), 1e-30), 0, 1)
    dist = np.linalg.norm(xy - (s + tt[..., None] * d), axis=-1)
    near = dist < 0.06
    keys = {"cost_pair_broad": c[:, 3], "cost_pair_narrow": c[:, 4] if c.shape[1] > 4 else c[:, 3],
            "near_count": near.sum(1).astype(np.float64),
            "near_polygons": (near & (table.kind != 0)).sum(1) * 16.0 + near.sum(1)}
    poly = table.kind != 0
    nv = np.where(poly, table.n_vertices, 0).astype(np.float64)
    for th in (0.03, 0.05, 0.12, 0.2):
        nr = dist < th
        keys[f"np16_{th}"] = (nr & poly).sum(1) * 16.0 + nr.sum(1)
    for th in (0.05, 0.08, 0.12):
        nr = dist < th
        keys[f"nvsum_{th}"] = (nr * nv).sum(1) + nr.sum(1)
        keys[f"nvsq_{th}"] = ((nr * nv).sum(1)) ** 2 + nr.sum(1)
    keys["all_polygons"] = poly.sum(1) * 16.0 + (dist < 0.08).sum(1)
    for name, key in keys.items():
        perm = np.argsort(-key, kind="stable")
        t = upload(perm)
        ms = time_it(t)
        res[name + "_desc"] = {"ms": ms, "speedup": res["orig_ms"] / ms, "bitwise_same_results": digest(t, perm) == d0}
        if name.startswith("cost"):
            res[name + "_corr_first"] = float(np.corrcoef(key, c[:, 3])[0, 1])
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
