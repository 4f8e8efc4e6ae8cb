"""TEST INFRASTRUCTURE ONLY: ctypes binding of oracle/liboracle.so, the plain-C
restatement of the reference hot path (oracle/pmbs_oracle.c).  Builds it with
gcc on first use when missing (gcc exists on the GPU box too)."""
from __future__ import annotations

import ctypes
import os
import subprocess
from ctypes import POINTER, c_double, c_int, c_int32, c_int64, c_uint64

import numpy as np

from paper_2207_06649_b200.abi import PpgParams, dptr, i64ptr, iptr, u64ptr
from paper_2207_06649_b200.world import ShapeTable, WorldState

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
_LIB = None


class OrcParams(ctypes.Structure):
    _fields_ = [("tip_r", c_double), ("tip_clear", c_double), ("push_distance", c_double),
                ("substeps", c_int), ("max_iters", c_int), ("eps_pen", c_double),
                ("rotation_gain", c_double), ("finger_width", c_double), ("finger_thickness", c_double),
                ("opening", c_double), ("approach_clearance", c_double), ("gamma", c_double),
                ("pushes_per_object", c_int), ("margin_threshold", c_double)]


def orc_params(p: PpgParams) -> OrcParams:
    return OrcParams(p.tip_radius, p.tip_clearance, p.push_distance, p.substeps, p.max_projection_iters,
                     p.eps_pen, p.rotation_gain, p.finger_width, p.finger_thickness, p.opening,
                     p.approach_clearance, p.gamma, p.pushes_per_object, p.margin_threshold)


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)


def lib():
    global _LIB
    if _LIB is None:
        src = os.path.join(HERE, "pmbs_oracle.c")
        if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(src):
            build()
        L = ctypes.CDLL(LIB)
        shape = [c_int, c_int, POINTER(c_int32), POINTER(c_double), POINTER(c_int32), POINTER(c_double),
                 POINTER(c_int32), c_double, c_double]
        L.orc_batch_resolve.argtypes = [c_int] + shape + [POINTER(c_double), POINTER(c_double),
                                                          POINTER(OrcParams), POINTER(c_double),
                                                          POINTER(c_int32), POINTER(c_double), POINTER(c_int64)]
        L.orc_state_digest.argtypes = [c_int] + shape + [POINTER(c_double), POINTER(c_uint64)]
        L.orc_sample_pushes.argtypes = [c_int] + shape + [POINTER(c_double), POINTER(OrcParams),
                                                          POINTER(c_double)]
        L.orc_graspable.argtypes = [c_int] + shape + [POINTER(c_double), POINTER(OrcParams), POINTER(c_double),
                                                      POINTER(c_double), POINTER(c_double), POINTER(c_int32)]
        L.orc_keyed_picks.argtypes = [c_uint64, c_uint64, c_uint64, c_int, c_uint64, POINTER(c_uint64)]
        L.orc_mix_keys.restype = c_uint64
        L.orc_mix_keys.argtypes = [c_uint64, c_uint64, c_uint64]
        L.orc_simulate.argtypes = shape + [POINTER(c_double), POINTER(c_int32), c_int, c_int, c_int, c_uint64,
                                           c_uint64, c_int, POINTER(OrcParams), POINTER(c_double),
                                           POINTER(c_int64)]
        _LIB = L
    return _LIB


def _shape_args(t: ShapeTable):
    return (t.n_objects, t.n_tables, iptr(t.kind), dptr(t.radius), iptr(t.n_vertices), dptr(t.vertices),
            iptr(t.target_index), t.side_length, t.boundary_margin)


def batch_resolve(table: ShapeTable, poses: np.ndarray, pushes: np.ndarray, params: PpgParams,
                  counts: bool = False):
    poses = np.ascontiguousarray(poses, np.float64)
    pushes = np.ascontiguousarray(pushes, np.float64)
    E = poses.shape[0]
    out = np.zeros_like(poses)
    status = np.zeros(E, np.int32)
    resid = np.zeros(E, np.float64)
    cnt = np.zeros((E, 8), np.int64) if counts else None
    op = orc_params(params)
    lib().orc_batch_resolve(E, *_shape_args(table), dptr(poses), dptr(pushes), ctypes.byref(op), dptr(out),
                            iptr(status), dptr(resid), i64ptr(cnt) if counts else None)
    return (out, status, resid, cnt) if counts else (out, status, resid)


def state_digests(table: ShapeTable, poses: np.ndarray) -> np.ndarray:
    poses = np.ascontiguousarray(poses, np.float64)
    out = np.zeros(poses.shape[0], np.uint64)
    lib().orc_state_digest(poses.shape[0], *_shape_args(table), dptr(poses), u64ptr(out))
    return out


def state_digest(st: WorldState) -> int:
    return int(state_digests(ShapeTable.shared(st), st.poses.reshape(1, st.n, 3))[0])


def sample_pushes(st: WorldState, params: PpgParams) -> np.ndarray:
    t = ShapeTable.shared(st)
    out = np.zeros((st.n * params.pushes_per_object, 4), np.float64)
    op = orc_params(params)
    k = lib().orc_sample_pushes(0, *_shape_args(t), dptr(np.ascontiguousarray(st.poses.reshape(1, st.n, 3))),
                                ctypes.byref(op), dptr(out))
    return out[:k].copy()


def graspable(st: WorldState, params: PpgParams):
    t = ShapeTable.shared(st)
    m = c_double()
    bx = c_double()
    by = c_double()
    bk = c_int32()
    op = orc_params(params)
    g = lib().orc_graspable(0, *_shape_args(t), dptr(np.ascontiguousarray(st.poses.reshape(1, st.n, 3))),
                            ctypes.byref(op), ctypes.byref(m), ctypes.byref(bx), ctypes.byref(by),
                            ctypes.byref(bk))
    return bool(g), m.value, bx.value, by.value, bk.value


def keyed_picks(seed: int, it: int, env: int, count: int, n: int) -> np.ndarray:
    out = np.zeros(count, np.uint64)
    lib().orc_keyed_picks(seed, it, env, count, n, u64ptr(out))
    return out


def mix_keys(seed: int, a: int, b: int = 0) -> int:
    return int(lib().orc_mix_keys(seed, a, b))


def simulate(scene: WorldState, node_poses: np.ndarray, node_meta: np.ndarray, n_envs: int, leaf_parallel: bool,
             seed: int, iteration: int, depth_cap: int, params: PpgParams):
    """batch_simulate / lockstep_simulate (pmbs.cpp:133-234) on given nodes."""
    t = ShapeTable.shared(scene)
    node_poses = np.ascontiguousarray(node_poses, np.float64)
    node_meta = np.ascontiguousarray(node_meta, np.int32)
    nn = node_poses.shape[0]
    rewards = np.zeros(nn, np.float64)
    ctr = np.zeros(4, np.int64)
    op = orc_params(params)
    rc = lib().orc_simulate(*_shape_args(t), dptr(node_poses), iptr(node_meta), nn, n_envs, 1 if leaf_parallel else 0,
                            seed, iteration, depth_cap, ctypes.byref(op), dptr(rewards), i64ptr(ctr))
    if rc != 0:
        raise ValueError("lockstep_simulate: fewer environments than nodes")
    return rewards, ctr
