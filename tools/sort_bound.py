"""Experiment: how much of the C2 kernel's lane idleness is env-cost mixing
inside a warp?  Times resolve_disc on the bench workload in its own order and
permuted by each env's MEASURED cost (the instrumented kernel's pair broad
tests: an oracle key no real launch has, so the upper bound of any
cost-grouping scheme) and by a cheap a-priori key.  Prints one JSON line.

    python tools/sort_bound.py [--envs 65536]
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
    ap.add_argument("--envs", type=int, default=65536)
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    import torch
    from paper_2207_06649_b200 import Context
    from paper_2207_06649_b200.abi import PpgShapes, default_params
    from paper_2207_06649_b200.scenes import c2_workload

    dev = torch.device("cuda", 0)
    ctx = Context(0, default_params())
    E, n = args.envs, 10
    table, poses, pushes, _ = c2_workload(ctx, E, n, 0.0)
    lib, stream = ctx.lib, torch.cuda.current_stream(dev)
    sptr = ctypes.c_void_p(stream.cuda_stream)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def upload(perm):
        t = dict(poses=torch.from_numpy(np.ascontiguousarray(poses[perm])).to(dev),
                 push=torch.from_numpy(np.ascontiguousarray(pushes[perm])).to(dev),
                 kind=torch.from_numpy(np.ascontiguousarray(table.kind[perm])).to(dev),
                 rad=torch.from_numpy(np.ascontiguousarray(table.radius[perm])).to(dev),
                 tgt=torch.from_numpy(np.ascontiguousarray(table.target_index[perm])).to(dev))
        t["out"] = torch.empty_like(t["poses"])
        t["st"] = torch.empty(E, dtype=torch.int32, device=dev)
        t["res"] = torch.empty(E, dtype=torch.float64, device=dev)
        t["sh"] = PpgShapes(n, E, ctypes.cast(t["kind"].data_ptr(), ctypes.POINTER(ctypes.c_int32)),
                            ctypes.cast(t["rad"].data_ptr(), ctypes.POINTER(ctypes.c_double)), None, None,
                            ctypes.cast(t["tgt"].data_ptr(), ctypes.POINTER(ctypes.c_int32)), 0.288, 0.0)
        return t

    def run(t):
        rc = lib.ppg_batch_resolve_dev(ctx.ptr, ctypes.byref(t["sh"]), t["poses"].data_ptr(), t["push"].data_ptr(),
                                       E, t["out"].data_ptr(), t["st"].data_ptr(), t["res"].data_ptr(), sptr)
        assert rc == 0, lib.ppg_last_error(ctx.ptr)

    def time_it(t):
        for _ in range(3):
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

    t0 = upload(np.arange(E))
    counts = torch.zeros((E, 8), dtype=torch.int64, device=dev)
    rc = lib.ppg_batch_resolve_count_dev(ctx.ptr, ctypes.byref(t0["sh"]), t0["poses"].data_ptr(),
                                         t0["push"].data_ptr(), E, counts.data_ptr(), sptr)
    assert rc == 0
    cost = counts.cpu().numpy()[:, 3].astype(np.float64)  # pair broad tests ~ projection iterations
    res = {"envs": E, "cost_mean": float(cost.mean()), "cost_p99": float(np.percentile(cost, 99)),
           "cost_max": float(cost.max())}
    w = cost[: E // 32 * 32].reshape(-1, 32)
    res["orig_warp_max_over_mean"] = float((w.max(1) / np.maximum(w.mean(1), 1)).mean())
    res["orig_ms"] = time_it(t0)
    torch.cuda.synchronize()
    ref_out = t0["out"].cpu().numpy()
    keys = {"oracle_cost_desc": np.argsort(-cost, kind="stable")}
    # a-priori key: discs near the push end (a second contact is likely)
    pe = pushes[:, 2:4]
    rad = np.asarray(table.radius, np.float64).reshape(E, -1)[:, :n]
    d = np.linalg.norm(poses[:, :, :2] - pe[:, None, :], axis=2) - rad
    keys["near_count_desc"] = np.argsort(-(d < 0.05).sum(1), kind="stable")
    res["near_key_cost_corr"] = float(np.corrcoef((d < 0.05).sum(1), cost)[0, 1])
    for name, perm in keys.items():
        t = upload(perm)
        ms = time_it(t)
        torch.cuda.synchronize()
        out = t["out"].cpu().numpy()
        inv = np.empty(E, np.int64)
        inv[perm] = np.arange(E)
        cp = cost[perm][: E // 32 * 32].reshape(-1, 32)
        res[name] = {"ms": ms, "speedup": res["orig_ms"] / ms,
                     "bitwise_same_results": bool(np.array_equal(out[inv], ref_out)),
                     "warp_max_over_mean": float((cp.max(1) / np.maximum(cp.mean(1), 1)).mean())}
        del t
    print(json.dumps(res))


if __name__ == "__main__":
    main()
