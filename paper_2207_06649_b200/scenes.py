"""Synthetic clutter inputs for the hot path (host side, no device needed).

``generate_cases`` restates the reference harness generators
(bench::generate_case / generate_case_motif, bench.cpp:234-317) in the C++
host library; ``keyed_picks`` restates keyed_rng + uniform_int_distribution
(rng.hpp:21-23, mcts.cpp:151-152).  ``c2_workload`` builds BASELINE.json
config 2: E scenes ``generate_case(10, ShapeMix{pf}, seed_base + k)`` with one
push each, ``sample_pushes(scene, 16)[pick(keyed_rng(7, k))]``.
"""
from __future__ import annotations

import os

import numpy as np

from . import abi
from .abi import dptr, iptr, u64ptr
from .world import ShapeTable, WorldState

MOTIFS = {"random": 0, "ring": 1, "wall": 2}


def generate_cases(n_objects: int, seeds, polygon_fraction: float = 0.0, motif: str = "random",
                   threads: int = 0):
    """Returns (ShapeTable with one table per scene, poses [E][n][3], ok [E])."""
    lib = abi.load_library()
    seeds = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64))
    E, n = len(seeds), n_objects
    kind = np.zeros((E, n), np.int32)
    radius = np.zeros((E, n), np.float64)
    nv = np.zeros((E, n), np.int32)
    verts = np.zeros((E, n, abi.PPG_MAX_VERTICES, 2), np.float64)
    poses = np.zeros((E, n, 3), np.float64)
    target = np.zeros(E, np.int32)
    ok = np.zeros(E, np.int32)
    rc = lib.ppg_generate_cases(MOTIFS[motif], n, polygon_fraction, u64ptr(seeds), E, iptr(kind), dptr(radius),
                                iptr(nv), dptr(verts), dptr(poses), iptr(target), iptr(ok),
                                threads or os.cpu_count() or 1)
    if rc != 0:
        raise ValueError("ppg_generate_cases: invalid arguments")
    return ShapeTable(kind, radius, nv, verts, target, 0.288, 0.0, n, E), poses, ok.astype(bool)


def generate_case(n_objects: int, polygon_fraction: float, seed: int, motif: str = "random") -> WorldState:
    t, poses, ok = generate_cases(n_objects, [seed], polygon_fraction, motif, threads=1)
    if not ok[0]:
        raise RuntimeError("generate_case: rejection sampling exhausted")
    return WorldState(t.kind[0].copy(), t.radius[0].copy(), t.n_vertices[0].copy(), t.vertices[0].copy(),
                      poses[0].copy(), int(t.target_index[0]), 0.288, 0.0)


def keyed_picks(seed: int, a, b, n) -> np.ndarray:
    lib = abi.load_library()
    n = np.ascontiguousarray(np.asarray(n, dtype=np.uint64))
    a = np.ascontiguousarray(np.broadcast_to(np.asarray(a, dtype=np.uint64), n.shape))
    b = np.ascontiguousarray(np.broadcast_to(np.asarray(b, dtype=np.uint64), n.shape))
    out = np.zeros(len(n), np.uint64)
    lib.ppg_keyed_picks(seed & 0xFFFFFFFFFFFFFFFF, u64ptr(a), u64ptr(b), u64ptr(n), len(n), u64ptr(out))
    return out


def c2_workload(ctx, E: int, n_objects: int = 10, polygon_fraction: float = 0.0, seed_base: int = 1000,
                pick_seed: int = 7):
    """BASELINE config 2 inputs.  Scenes whose generator throws or that have
    no legal push are replaced by the next seed (rare).  Pushes are sampled on
    the device (ppg_sample_pushes, per-env shapes) and picked on the host."""
    seeds = np.arange(seed_base, seed_base + int(E * 1.05) + 64, dtype=np.uint64)
    table, poses, ok = generate_cases(n_objects, seeds, polygon_fraction)
    sel = np.nonzero(ok)[0]
    table = _take(table, sel)
    poses = poses[sel]
    seeds = seeds[sel]
    cand, cnt = ctx.sample_pushes_arrays(poses, table)
    sel = np.nonzero(cnt > 0)[0][:E]
    if len(sel) < E:
        raise RuntimeError("c2_workload: not enough valid scenes")
    table, poses, seeds, cand, cnt = _take(table, sel), poses[sel], seeds[sel], cand[sel], cnt[sel]
    k = np.arange(E, dtype=np.uint64)
    pick = keyed_picks(pick_seed, k, 0, cnt.astype(np.uint64)).astype(np.int64)
    pushes = np.ascontiguousarray(cand[np.arange(E), pick])
    return table, np.ascontiguousarray(poses), pushes, seeds


def _take(t: ShapeTable, idx) -> ShapeTable:
    return ShapeTable(np.ascontiguousarray(t.kind[idx]), np.ascontiguousarray(t.radius[idx]),
                      np.ascontiguousarray(t.n_vertices[idx]), np.ascontiguousarray(t.vertices[idx]),
                      np.ascontiguousarray(t.target_index[idx]), t.side_length, t.boundary_margin, t.n_objects,
                      len(idx))
