"""Generates the golden fixtures in tests/golden/ from the UNMODIFIED reference
(oracle/_ref/libpushplan_ref.so, built from /root/reference by oracle/Makefile).

    python tests/golden/make_golden.py        # needs oracle/_ref (this container)

Fixtures (all values produced by the reference's own public API):
  cases.json        the 20 proj/cases scenes as loaded by load_scene
                    (world.cpp:271-277), their state_digest, sample_pushes
                    count + FNV of the action bytes, graspable report, and the
                    first PMBS decision at the reference defaults (N_e = 64,
                    seed = mix_keys(episode_seed(0, case, 0), 0), bench.cpp:50-52, 95):
                    action, iterations, expansions, stop reason, final d_T,
                    FNV-1a of tree_signature.
  resolve_*.npz     batch_resolve (push_sim.cpp:132-152) on generate_case
                    scenes (bench.cpp:234-259) with a keyed sampled push:
                    inputs + status + state digests + residual-free outputs.
  simulate.npz      first-iteration children of several cases and the
                    reference batch_simulate rewards (pmbs.cpp:207-234).
  rng.json          keyed_rng + uniform_int_distribution picks (rng.hpp:21-23,
                    mcts.cpp:151-152).
"""
import glob
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from paper_2207_06649_b200.abi import default_params  # noqa: E402
from paper_2207_06649_b200.world import ShapeTable  # noqa: E402

CASES = "/root/reference/proj/cases"


def fnv_bytes(b: bytes) -> int:
    h = 1469598103934665603
    for c in b:
        h ^= c
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def state_json(s):
    return {"kind": s.kind.tolist(), "radius": s.radius.tolist(), "n_vertices": s.n_vertices.tolist(),
            "vertices": s.vertices.tolist(), "poses": s.poses.tolist(), "target_index": s.target_index,
            "side_length": s.side_length, "boundary_margin": s.boundary_margin}


def cases():
    p = default_params()
    out = []
    for f in sorted(glob.glob(os.path.join(CASES, "*.json"))):
        cid = os.path.splitext(os.path.basename(f))[0]
        s = ref.load_scene(f)
        sp = ref.sample_pushes(s, p)
        g = ref.graspable(s, p)
        seed = ref.mix_keys(ref.episode_seed(0, cid, 0), 0)
        q = default_params(rng_seed=seed)
        r = ref.run_search(s, q, threads=1)
        out.append({"case_id": cid, "state": state_json(s), "digest": str(ref.state_digest(s)),
                    "n_pushes": int(len(sp)), "pushes_fnv": str(fnv_bytes(sp.tobytes())),
                    "graspable": g[0], "margin": g[1], "best": [g[2], g[3], g[4]],
                    "seed": str(seed),
                    "decision": {"action": r["action"].tolist(), "iterations": r["iterations"],
                                 "expansions": r["expansions"], "stop": r["stop"],
                                 "final_tree_depth": r["final_tree_depth"], "sig_fnv": str(r["sig_fnv"]),
                                 "n_nodes": r["n_nodes"]}})
        print(cid, r["iterations"], r["expansions"], r["stop"], hex(r["sig_fnv"]), flush=True)
    with open(os.path.join(HERE, "cases.json"), "w") as fh:
        json.dump(out, fh)


def resolve_set(name, polygon_fraction, count, seed0, n_objects=10, motif=0, per_scene=1):
    p = default_params()
    states, pushes = [], []
    k = 0
    while len(states) < count:
        try:
            s = ref.generate_case(n_objects, polygon_fraction, seed0 + k, motif)
        except RuntimeError:  # BenchError: rejection sampling exhausted
            k += 1
            continue
        sp = ref.sample_pushes(s, p)
        for j in range(min(per_scene, len(sp))):
            pick = int(ref.keyed_picks(7, seed0 + k, j, 1, len(sp))[0])
            states.append(s)
            pushes.append(sp[pick])
        k += 1
    states, pushes = states[:count], pushes[:count]
    t = ShapeTable.per_env(states)
    P = np.stack([s.poses for s in states])
    A = np.stack(pushes)
    out, status, dig, _ = ref.batch_resolve(t, P, A, p, threads=8)
    np.savez_compressed(os.path.join(HERE, f"resolve_{name}.npz"), kind=t.kind, radius=t.radius,
                        n_vertices=t.n_vertices, vertices=t.vertices, target=t.target_index, poses=P, pushes=A,
                        status=status, digests=dig, out=out)
    print(name, "status counts", np.bincount(status, minlength=3), flush=True)


def hard_set(count_bad=160, count_ok=240):
    """Depth-2 states of dense ring scenes (generate_case_motif Ring, 18
    objects): every sampled push, keeping the non-converged ones (SimError,
    push_sim.cpp:123-128) and a sample of converged ones."""
    p = default_params()
    states, pushes = [], []
    nb = no = 0
    k = 0
    while nb < count_bad or no < count_ok:
        k += 1
        try:
            s = ref.generate_case(18, 0.0, 7000 + k, 1)
        except RuntimeError:
            continue
        sp = ref.sample_pushes(s, p)
        t = ShapeTable.shared(s)
        out, st, _, _ = ref.batch_resolve(t, np.repeat(s.poses[None], len(sp), 0), sp, p, threads=8)
        for j in np.nonzero(st == 0)[0][:12]:
            s2 = s.with_poses(out[j])
            sp2 = ref.sample_pushes(s2, p)
            if len(sp2) == 0:
                continue
            _, st2, _, _ = ref.batch_resolve(ShapeTable.shared(s2), np.repeat(s2.poses[None], len(sp2), 0), sp2,
                                             p, threads=8)
            for q in range(len(sp2)):
                if st2[q] != 0 and nb < count_bad:
                    states.append(s2)
                    pushes.append(sp2[q])
                    nb += 1
                elif st2[q] == 0 and no < count_ok and q % 7 == 0:
                    states.append(s2)
                    pushes.append(sp2[q])
                    no += 1
    t = ShapeTable.per_env(states)
    P = np.stack([s.poses for s in states])
    A = np.stack(pushes)
    out, status, dig, _ = ref.batch_resolve(t, P, A, p, threads=8)
    np.savez_compressed(os.path.join(HERE, "resolve_hard18.npz"), kind=t.kind, radius=t.radius,
                        n_vertices=t.n_vertices, vertices=t.vertices, target=t.target_index, poses=P, pushes=A,
                        status=status, digests=dig, out=out)
    print("hard18 status counts", np.bincount(status, minlength=3), flush=True)


def simulate():
    res = {}
    for cid, ne, seed in [("case_13", 64, 11), ("case_18", 64, 12), ("case_11", 200, 13), ("case_16", 64, 14),
                          ("case_20", 128, 15)]:
        s = ref.load_scene(os.path.join(CASES, cid + ".json"))
        p = default_params(n_envs=ne, rng_seed=seed)
        poses, meta, rew, cap = ref.first_iteration(s, p, 0)
        res[f"{cid}_{ne}_poses"] = poses
        res[f"{cid}_{ne}_meta"] = meta
        res[f"{cid}_{ne}_rewards"] = rew
        res[f"{cid}_{ne}_cap"] = np.array([cap, seed, ne])
        print(cid, ne, len(rew), rew.max(), flush=True)
    np.savez_compressed(os.path.join(HERE, "simulate.npz"), **res)


def rng():
    out = []
    for seed, it, env, n in [(0, 0, 0, 17), (7, 3, 1000, 160), (12345, 99, 63, 1), (2 ** 63 + 5, 7, 5, 3),
                             (42, 0, 7, 2 ** 40 + 3)]:
        out.append({"seed": str(seed), "iter": it, "env": env, "n": str(n),
                    "picks": [str(v) for v in ref.keyed_picks(seed, it, env, 400, n)],
                    "raw": [str(v) for v in ref.keyed_raw(seed, it, env, 700)]})
    with open(os.path.join(HERE, "rng.json"), "w") as fh:
        json.dump(out, fh)


def acceptance():
    """Reference acceptance criteria C1 (acceptance.cpp:184-211: N_e = 1 PMBS
    == serial MCTS on 25 deep cases x 500 iterations) and C4 (:283-305:
    N_e = 16, 200 iterations, identical across pool sizes) — the expected
    trees (FNV of tree_signature) and actions from the reference."""
    out = {"c1": [], "c4": []}
    for i in range(25):
        st = ref.deep_search_case(1000 + i, 8 + i % 5)
        p = default_params(budget_iterations=1, max_iterations=500, rng_seed=4000 + i)
        r = ref.run_search(st, p, threads=1, serial=True)
        q = ref.run_search(st, default_params(budget_iterations=1, max_iterations=500, rng_seed=4000 + i, n_envs=1,
                                              leaf_parallel=0), threads=1)
        assert q["sig_fnv"] == r["sig_fnv"]
        out["c1"].append({"state": state_json(st), "seed": 4000 + i, "sig_fnv": str(r["sig_fnv"]),
                          "action": r["action"].tolist(), "iterations": r["iterations"], "stop": r["stop"]})
    for i in range(10):
        st = ref.deep_search_case(2000 + i, 8 + i % 5)
        p = default_params(budget_iterations=1, max_iterations=200, rng_seed=500 + i, n_envs=16)
        r = ref.run_search(st, p, threads=8)
        out["c4"].append({"state": state_json(st), "seed": 500 + i, "sig_fnv": str(r["sig_fnv"]),
                          "action": r["action"].tolist(), "iterations": r["iterations"], "stop": r["stop"]})
    with open(os.path.join(HERE, "acceptance.json"), "w") as fh:
        json.dump(out, fh)
    print("acceptance c1/c4", len(out["c1"]), len(out["c4"]), flush=True)


def c3():
    """Acceptance criterion 3 (acceptance.cpp:255-281): 200 random explicit
    trees and the reference select_batch's pairs / virtual visits (variant 0
    = the criterion exactly; variant 1 adds terminal nodes and d_T 1-4)."""
    res = {}
    for v in (0, 1):
        a = ref.c3_trees(v)
        for k, x in a.items():
            res[f"v{v}_{k}"] = x
        print("c3 variant", v, "nodes", a["node_off"][-1], "pairs", a["pair_off"][-1], flush=True)
    np.savez_compressed(os.path.join(HERE, "c3_trees.npz"), **res)


def _decision(st, p, threads=8):
    r = ref.run_search(st, p, threads=threads)
    return {"action": r["action"].tolist(), "iterations": r["iterations"], "expansions": r["expansions"],
            "stop": r["stop"], "final_tree_depth": r["final_tree_depth"], "sig_fnv": str(r["sig_fnv"]),
            "n_nodes": r["n_nodes"]}


WIDE_16K = [("case_13", 16384), ("case_18", 16384)]


def wide():
    """Reference run_pmbs fingerprints beyond the defaults (VERDICT r1 task 1):
    case_18 / case_13 at N_e 1000 / 4096 (case_13 at 1000 draws past the
    156-word MT19937-64 block), C4 dense ring motifs (ring-16 / ring-18, seeds
    5 and 19, d_T 9, N_a 24, N_e 4096, 10 iterations) and the polygon cases
    16 / 17 at N_e 1000.  Iteration budgets (not seconds) keep every run
    machine-independent."""
    out = []
    cs = {}
    for f in sorted(glob.glob(os.path.join(CASES, "*.json"))):
        cs[os.path.splitext(os.path.basename(f))[0]] = f
    with open(os.path.join(HERE, "cases.json")) as fh:
        seeds = {c["case_id"]: int(c["seed"]) for c in json.load(fh)}
    runs = [("case_18", 1000), ("case_18", 4096), ("case_13", 1000), ("case_13", 4096), ("case_16", 1000),
            ("case_17", 1000)] + WIDE_16K
    for cid, ne in runs:
        st = ref.load_scene(cs[cid])
        p = default_params(rng_seed=seeds[cid], n_envs=ne, budget_iterations=1, max_iterations=200)
        d = _decision(st, p)
        out.append({"kind": "case", "case_id": cid, "n_envs": ne, "seed": str(seeds[cid]), "max_iterations": 200,
                    "decision": d})
        print(cid, ne, d["iterations"], d["stop"], flush=True)
    for n in (16, 18):
        for seed in (5, 19):
            st = ref.generate_case(n, 0.0, seed, 1)
            p = default_params(rng_seed=seed, n_envs=4096, tree_depth=9, pushes_per_object=24, budget_iterations=1,
                               max_iterations=10)
            d = _decision(st, p)
            out.append({"kind": "ring", "n_objects": n, "scene_seed": seed, "seed": str(seed), "n_envs": 4096,
                        "tree_depth": 9, "pushes_per_object": 24, "max_iterations": 10, "decision": d})
            print("ring", n, seed, d["iterations"], d["stop"], flush=True)
    with open(os.path.join(HERE, "wide.json"), "w") as fh:
        json.dump(out, fh, indent=0)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        globals()[sys.argv[1]]()
        sys.exit(0)
    rng()
    cases()
    resolve_set("discs", 0.0, 384, 1000)
    resolve_set("polygons", 0.35, 256, 50000)
    resolve_set("ring16", 0.0, 512, 90000, n_objects=16, motif=1, per_scene=16)
    hard_set()
    simulate()
