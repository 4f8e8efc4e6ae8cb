"""Randomised parity stress of the device-tree search (asynchronous lockstep
with early, pending-bound and speculative decisions) against the unmodified
reference (oracle/_ref): random generated scenes (discs and polygon mixes,
random / ring / wall motifs), several seeds and N_e; every decision's action,
tree signature and work counters must match.
    python tools/stress_decisions.py [count]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402
from paper_2207_06649_b200 import Context, ParallelConfig, run_pmbs  # noqa: E402
from paper_2207_06649_b200.scenes import generate_case  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 40
ctx = Context(0)
threads = os.cpu_count() or 1
bad, done = [], 0
motifs = ["random", "ring", "wall"]
for k in range(count):
    n = 6 + (k * 7) % 11
    pf = [0.0, 0.0, 0.35, 1.0][k % 4]
    if pf > 0 and n > 16:
        n = 12
    motif = motifs[k % 3]
    seed = 1000 + 37 * k
    try:
        st = generate_case(n, pf, seed, motif)
    except RuntimeError:
        continue
    for ne in (64, 256) if k % 2 == 0 else (64, 1000):
        cfg = ParallelConfig(rng_seed=seed, n_envs=ne)
        try:
            r = run_pmbs(st, cfg, ctx=ctx)
        except Exception as ex:  # noqa: BLE001
            q = ref.run_search(st, cfg.to_params(), threads=threads)
            if q.get("rc", 0) == 0:
                bad.append((k, ne, "device error: " + str(ex)))
            continue
        q = ref.run_search(st, cfg.to_params(), threads=threads)
        same = (list(q["action"]) == list(r.action) and q["sig_fnv"] == r.signature_fnv)
        done += 1
        if not same:
            bad.append((k, ne, n, pf, motif))
print(json.dumps({"decisions": done, "mismatches": bad}))
