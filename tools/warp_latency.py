"""Latency mode (one warp per environment): device latency of ONE
environment's resolve_push per projection iteration.

For the golden resolve sets, the environments with the most projection
iterations (counted by the oracle: iterations = tip broad tests / active
objects) are replicated 148x (one warp per SM, so the call time is one
environment's latency) and timed through ppg_batch_resolve.  Prints one JSON
line per environment and a summary (ns per iteration)."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import golden_io  # noqa: E402
from oracle import port  # noqa: E402
from paper_2207_06649_b200 import Context, default_params  # noqa: E402
from paper_2207_06649_b200.scenes import _take  # noqa: E402


def main():
    P = default_params()
    ctx = Context(0, P)
    rows = []
    for name in sys.argv[1:] or ["discs", "hard18", "ring16"]:
        t, poses, pushes, status, dig, out = golden_io.resolve_set(name)
        _, s, _, c = port.batch_resolve(t, poses, pushes, P, counts=True)
        tb, pb = c[:, 0].astype(np.float64), c[:, 3].astype(np.float64)
        act = np.where(tb > 0, 2 * pb / np.maximum(tb, 1) + 1, 1)
        iters = np.where(tb > 0, tb / act, 0)
        hits = c[:, 5].astype(np.float64)
        order = np.argsort(-iters)
        for k in order[:6].tolist():
            if iters[k] < 200:
                continue
            R = 148
            sel = np.full(R, k)
            tt = _take(t, sel)
            pp = np.ascontiguousarray(poses[sel])
            aa = np.ascontiguousarray(pushes[sel])
            ctx.batch_resolve_arrays(tt, pp, aa)
            best = 1e9
            for _ in range(5):
                t0 = time.perf_counter()
                ctx.batch_resolve_arrays(tt, pp, aa)
                best = min(best, time.perf_counter() - t0)
            r = {"set": name, "env": k, "n": int(poses.shape[1]), "status": int(s[k]), "iterations": int(iters[k]),
                 "pair_hits": int(hits[k]), "us": best * 1e6, "ns_per_iter": best * 1e9 / iters[k],
                 "ns_per_hit": best * 1e9 / max(1, hits[k])}
            rows.append(r)
            print(json.dumps(r), flush=True)
    it = sum(r["iterations"] for r in rows)
    us = sum(r["us"] for r in rows)
    print(json.dumps({"summary": True, "envs": len(rows), "ns_per_iter": us * 1e3 / max(1, it)}))
    ctx.close()


if __name__ == "__main__":
    main()
