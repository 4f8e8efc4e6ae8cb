"""A reduced parity subset for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): the streamed host batch_resolve (ready flags,
zero-copy outputs), the device-resident tree on case_18 (graph with the
lockstep WHILE node), latency-mode polygon batches, the lane-mode disc
kernel, and the emulated multi-shard lockstep — each checked bitwise against
the oracle / reference goldens so a sanitizer run is also a parity run.

    compute-sanitizer --tool memcheck python tools/sanitize_subset.py [quick]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import golden_io  # noqa: E402
from oracle import port  # noqa: E402
from paper_2207_06649_b200 import Context, ParallelConfig, default_params, run_pmbs  # noqa: E402
from paper_2207_06649_b200.scenes import _take, c2_workload  # noqa: E402

quick = len(sys.argv) > 1 and sys.argv[1] == "quick"
P = default_params()
ctx = Context(0, P)
# 1. streamed host batch_resolve (>= 32K envs), pinned outputs (zero-copy), start collisions included
E = 32784
table, poses, pushes, _ = c2_workload(ctx, E)
pushes = pushes.copy()
hit = np.arange(5, E, 501)
pushes[hit, 0:2] = poses[hit, 0, 0:2]
pushes[hit, 2:4] = poses[hit, 0, 0:2] + 0.05
import torch  # noqa: E402
po = torch.empty(poses.shape, dtype=torch.float64).pin_memory().numpy()
ps = torch.empty((E,), dtype=torch.int32).pin_memory().numpy()
pr = torch.empty((E,), dtype=torch.float64).pin_memory().numpy()
ctx.batch_resolve_arrays(table, poses, pushes, out=(po, ps, pr))
idx = np.linspace(0, E - 1, 300).astype(np.int64)
o3, s3, _ = port.batch_resolve(_take(table, idx), np.ascontiguousarray(poses[idx]), np.ascontiguousarray(pushes[idx]), P)
assert np.array_equal(ps[idx], s3) and np.array_equal(po[idx].view(np.uint64), o3.view(np.uint64))
print("streamed zero-copy batch_resolve ok", flush=True)
# 2. lane-mode disc kernel + latency-mode polygons on the golden sets
for name in ("discs", "polygons"):
    t, p, a, status, digests, _ = golden_io.resolve_set(name)
    k = 128 if quick else len(status)
    out, st, _ = ctx.batch_resolve_arrays(_take(t, np.arange(k)), p[:k], a[:k])
    assert np.array_equal(st, status[:k])
    assert np.array_equal(port.state_digests(_take(t, np.arange(k)), out)[st == 0], digests[:k][st == 0])
    print(name, "golden batch ok", flush=True)
# 3. device tree decisions (graph + WHILE node): case_18 and a polygon case
cases = golden_io.cases()
for idx_case in ((17,) if quick else (17, 15)):
    cc, st = cases[idx_case]
    r = run_pmbs(st, ParallelConfig(rng_seed=int(cc["seed"])), ctx=ctx)
    assert r.signature_fnv == int(cc["decision"]["sig_fnv"]), cc["case_id"]
    print(cc["case_id"], "decision ok", flush=True)
ctx.close()
# 4. emulated 2-shard lockstep + sharded decision
m = Context.multi([0, 0], emulate=True)
cc, st = cases[12]
r = run_pmbs(st, ParallelConfig(rng_seed=int(cc["seed"])), ctx=m)
assert r.signature_fnv == int(cc["decision"]["sig_fnv"])
m.close()
print("sharded decision ok", flush=True)
print("SANITIZE SUBSET OK")
