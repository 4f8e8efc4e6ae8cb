"""Loaders for the committed golden fixtures (tests/golden/, made by
tests/golden/make_golden.py from the unmodified reference)."""
import json
import os

import numpy as np

from paper_2207_06649_b200.world import ShapeTable, WorldState

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def cases():
    with open(os.path.join(GOLDEN, "cases.json")) as f:
        data = json.load(f)
    out = []
    for c in data:
        s = c["state"]
        st = WorldState(np.array(s["kind"], np.int32), np.array(s["radius"], np.float64),
                        np.array(s["n_vertices"], np.int32), np.array(s["vertices"], np.float64),
                        np.array(s["poses"], np.float64), s["target_index"], s["side_length"],
                        s["boundary_margin"])
        out.append((c, st))
    return out


def resolve_set(name):
    z = np.load(os.path.join(GOLDEN, f"resolve_{name}.npz"))
    E, n = z["poses"].shape[:2]
    t = ShapeTable(np.ascontiguousarray(z["kind"]), np.ascontiguousarray(z["radius"]),
                   np.ascontiguousarray(z["n_vertices"]), np.ascontiguousarray(z["vertices"]),
                   np.ascontiguousarray(z["target"]), 0.288, 0.0, n, E)
    return t, np.ascontiguousarray(z["poses"]), np.ascontiguousarray(z["pushes"]), z["status"], z["digests"], z["out"]


RESOLVE_SETS = ["discs", "polygons", "ring16", "hard18"]


def simulate_sets():
    z = np.load(os.path.join(GOLDEN, "simulate.npz"))
    keys = sorted({k.rsplit("_", 1)[0] for k in z.files})
    out = []
    for k in keys:
        cid = "_".join(k.split("_")[:2])
        cap, seed, ne = (int(v) for v in z[k + "_cap"])
        out.append((cid, ne, seed, cap, z[k + "_poses"], z[k + "_meta"], z[k + "_rewards"]))
    return out


def rng():
    with open(os.path.join(GOLDEN, "rng.json")) as f:
        return json.load(f)


def fnv_bytes(b: bytes) -> int:
    h = 1469598103934665603
    for c in b:
        h ^= c
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def _state(s):
    return WorldState(np.array(s["kind"], np.int32), np.array(s["radius"], np.float64),
                      np.array(s["n_vertices"], np.int32), np.array(s["vertices"], np.float64),
                      np.array(s["poses"], np.float64), s["target_index"], s["side_length"], s["boundary_margin"])


def acceptance():
    """Reference acceptance C1 / C4 fixtures (tests/golden/make_golden.py acceptance)."""
    with open(os.path.join(GOLDEN, "acceptance.json")) as f:
        d = json.load(f)
    return {k: [(x, _state(x["state"])) for x in v] for k, v in d.items()}


def c3_trees(variant: int):
    """Acceptance C3 fixture: random explicit trees + the reference select_batch."""
    z = np.load(os.path.join(GOLDEN, "c3_trees.npz"))
    return {k[len(f"v{variant}_"):]: z[k] for k in z.files if k.startswith(f"v{variant}_")}


def wide():
    """Reference run_pmbs fingerprints at wide N_e / C4 / polygon cases."""
    with open(os.path.join(GOLDEN, "wide.json")) as f:
        return json.load(f)
