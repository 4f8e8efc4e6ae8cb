"""TEST INFRASTRUCTURE ONLY: ctypes binding of oracle/_ref/libpushplan_ref.so,
the unmodified reference (arxiv 2207.06649 pushplan core) + oracle/ref_shim.cpp."""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_int32, c_int64, c_uint64, c_void_p

import numpy as np

from paper_2207_06649_b200.abi import (PPG_MAX_VERTICES, PpgParams, PpgSearchStats, PpgShapes,
                                       STOP_REASONS, dptr, i64ptr, iptr, u64ptr)
from paper_2207_06649_b200.world import ShapeTable, WorldState

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "libpushplan_ref.so")
_LIB = None


def available() -> bool:
    return os.path.exists(REF_LIB)


def lib():
    global _LIB
    if _LIB is None:
        if not available():
            raise RuntimeError(f"{REF_LIB} missing (build with `make -C oracle ref` where /root/reference exists)")
        L = ctypes.CDLL(REF_LIB)
        L.ref_states_new.restype = c_void_p
        L.ref_states_new.argtypes = [POINTER(PpgShapes), POINTER(c_double), c_int]
        L.ref_states_free.argtypes = [c_void_p]
        L.ref_state_n.argtypes = [c_void_p, c_int]
        L.ref_state_export.argtypes = [c_void_p, c_int, POINTER(c_int32), POINTER(c_double), POINTER(c_int32),
                                       POINTER(c_double), POINTER(c_double), POINTER(c_int32),
                                       POINTER(c_double), POINTER(c_double)]
        L.ref_generate_case.restype = c_void_p
        L.ref_generate_case.argtypes = [c_int, c_int, c_double, c_uint64]
        L.ref_c2_workload.restype = c_void_p
        L.ref_c2_workload.argtypes = [c_int, c_double, c_uint64, c_int, c_uint64, c_int, c_int, POINTER(c_double),
                                      POINTER(c_uint64)]
        L.ref_c3_trees.argtypes = [c_int, c_int, c_int, c_int] + [c_void_p] * 16
        L.ref_batch_simulate.argtypes = [c_void_p, POINTER(c_int32), c_int, POINTER(PpgParams), c_uint64, c_int, c_int,
                                         POINTER(c_double), POINTER(c_double)]
        L.ref_load_scene.restype = c_void_p
        L.ref_load_scene.argtypes = [c_char_p]
        L.ref_fixture.restype = c_void_p
        L.ref_fixture.argtypes = [c_char_p, c_double, c_int]
        L.ref_deep_search_case.restype = c_void_p
        L.ref_deep_search_case.argtypes = [c_uint64, c_int]
        L.ref_state_digest.restype = c_uint64
        L.ref_state_digest.argtypes = [c_void_p, c_int]
        L.ref_batch_resolve.argtypes = [c_void_p, POINTER(c_double), POINTER(PpgParams), c_int, POINTER(c_double)]
        L.ref_batch_results.argtypes = [c_void_p, POINTER(c_double), POINTER(c_int32), POINTER(c_uint64)]
        L.ref_sample_pushes.argtypes = [c_void_p, c_int, POINTER(PpgParams), POINTER(c_double), c_int]
        L.ref_graspable.argtypes = [c_void_p, c_int, POINTER(PpgParams), POINTER(c_double), POINTER(c_double),
                                    POINTER(c_double), POINTER(c_int32)]
        L.ref_keyed_picks.argtypes = [c_uint64, c_uint64, c_uint64, c_int, c_uint64, POINTER(c_uint64)]
        L.ref_keyed_raw.argtypes = [c_uint64, c_uint64, c_uint64, c_int, POINTER(c_uint64)]
        L.ref_mix_keys.restype = c_uint64
        L.ref_mix_keys.argtypes = [c_uint64, c_uint64, c_uint64]
        L.ref_episode_seed.restype = c_uint64
        L.ref_episode_seed.argtypes = [c_uint64, c_char_p, c_int]
        L.ref_run_search.argtypes = [c_void_p, c_int, POINTER(PpgParams), c_int, c_int, POINTER(c_double),
                                     POINTER(PpgSearchStats), c_char_p, c_int64, POINTER(c_int64)]
        L.ref_first_iteration.argtypes = [c_void_p, c_int, POINTER(PpgParams), c_uint64, POINTER(c_double),
                                          POINTER(c_int32), POINTER(c_double), POINTER(c_int32)]
        L.ref_run_episode.argtypes = [c_void_p, c_int, c_char_p, c_int, POINTER(PpgParams), c_int, c_uint64,
                                      c_int, POINTER(c_int32), POINTER(c_double), c_char_p]
        L.ref_replay_log.argtypes = [c_char_p, c_char_p, c_int]
        _LIB = L
    return _LIB


class Handle:
    """Owns a std::vector<WorldState> inside the reference library."""

    def __init__(self, ptr):
        if not ptr:
            raise RuntimeError("reference call failed")
        self.ptr = ptr

    def __del__(self):
        if getattr(self, "ptr", None) and _LIB is not None:
            _LIB.ref_states_free(self.ptr)
            self.ptr = None

    def export(self, i: int = 0) -> WorldState:
        L = lib()
        n = L.ref_state_n(self.ptr, i)
        kind = np.zeros(n, np.int32)
        radius = np.zeros(n, np.float64)
        nv = np.zeros(n, np.int32)
        verts = np.zeros((n, PPG_MAX_VERTICES, 2), np.float64)
        poses = np.zeros((n, 3), np.float64)
        tgt = c_int32()
        side = c_double()
        margin = c_double()
        L.ref_state_export(self.ptr, i, iptr(kind), dptr(radius), iptr(nv), dptr(verts), dptr(poses),
                           ctypes.byref(tgt), ctypes.byref(side), ctypes.byref(margin))
        return WorldState(kind, radius, nv, verts, poses, tgt.value, side.value, margin.value)


def states_handle(table: ShapeTable, poses: np.ndarray) -> Handle:
    poses = np.ascontiguousarray(poses, np.float64)
    E = poses.shape[0]
    return Handle(lib().ref_states_new(ctypes.byref(table.struct()), dptr(poses), E))


def state_handle(st: WorldState) -> Handle:
    return states_handle(ShapeTable.shared(st), st.poses.reshape(1, st.n, 3))


def generate_case(n_objects: int, polygon_fraction: float, seed: int, motif: int = 0) -> WorldState:
    """bench::generate_case / generate_case_motif (bench.cpp:234-317)."""
    h = Handle(lib().ref_generate_case(motif, n_objects, polygon_fraction, seed))
    return h.export(0)


def load_scene(path: str) -> WorldState:
    h = Handle(lib().ref_load_scene(path.encode()))
    return h.export(0)


def fixture(name: str, arg: float = 0.0, iarg: int = 0) -> WorldState:
    """tests/support/scenes.cpp fixtures."""
    h = Handle(lib().ref_fixture(name.encode(), arg, iarg))
    return h.export(0)


def deep_search_case(seed: int, n_objects: int) -> WorldState:
    """acceptance.cpp:124-134."""
    h = Handle(lib().ref_deep_search_case(seed, n_objects))
    return h.export(0)


def state_digest(st: WorldState) -> int:
    h = state_handle(st)
    return int(lib().ref_state_digest(h.ptr, 0))


def batch_resolve(table: ShapeTable, poses: np.ndarray, pushes: np.ndarray, params: PpgParams,
                  threads: int = 1):
    """pushplan::batch_resolve (push_sim.cpp:132-152).  Returns poses_out,
    status, digests, seconds (the reference call alone)."""
    h = states_handle(table, poses)
    pushes = np.ascontiguousarray(pushes, np.float64)
    secs = c_double()
    lib().ref_batch_resolve(h.ptr, dptr(pushes), ctypes.byref(params), threads, ctypes.byref(secs))
    E = poses.shape[0]
    out = np.zeros_like(np.ascontiguousarray(poses, np.float64))
    status = np.zeros(E, np.int32)
    dig = np.zeros(E, np.uint64)
    lib().ref_batch_results(h.ptr, dptr(out), iptr(status), u64ptr(dig))
    return out, status, dig, secs.value


def c2_workload(E: int, n_objects: int = 10, polygon_fraction: float = 0.0, seed_base: int = 1000,
                pick_seed: int = 7, pushes_per_object: int = 16, threads: int = 0):
    """BASELINE config 2 inputs built by the reference alone
    (bench::generate_case + sample_pushes + keyed pick; ref_shim.cpp
    ref_c2_workload).  Returns (Handle of E states, pushes [E][4], seeds [E])."""
    pushes = np.zeros((E, 4), np.float64)
    seeds = np.zeros(E, np.uint64)
    ptr = lib().ref_c2_workload(n_objects, polygon_fraction, seed_base, E, pick_seed, pushes_per_object,
                                threads or os.cpu_count() or 1, dptr(pushes), u64ptr(seeds))
    return Handle(ptr), pushes, seeds


class PreparedBatch:
    """States built once; ``run`` times only pushplan::batch_resolve."""

    def __init__(self, table: ShapeTable, poses: np.ndarray, pushes: np.ndarray, params: PpgParams,
                 handle=None):
        self.h = handle if handle is not None else states_handle(table, poses)
        self.pushes = np.ascontiguousarray(pushes, np.float64)
        self.params = params
        self.E = len(self.pushes)

    def run(self, threads: int) -> float:
        secs = c_double()
        lib().ref_batch_resolve(self.h.ptr, dptr(self.pushes), ctypes.byref(self.params), threads,
                                ctypes.byref(secs))
        return secs.value

    def results(self, n_objects: int):
        """(poses_out [E][n][3], status [E], digests [E]) of the last run."""
        out = np.zeros((self.E, n_objects, 3), np.float64)
        status = np.zeros(self.E, np.int32)
        dig = np.zeros(self.E, np.uint64)
        lib().ref_batch_results(self.h.ptr, dptr(out), iptr(status), u64ptr(dig))
        return out, status, dig


def sample_pushes(st: WorldState, params: PpgParams) -> np.ndarray:
    h = state_handle(st)
    cap = st.n * params.pushes_per_object
    out = np.zeros((cap, 4), np.float64)
    k = lib().ref_sample_pushes(h.ptr, 0, ctypes.byref(params), dptr(out), cap)
    return out[:k].copy()


def graspable(st: WorldState, params: PpgParams):
    h = state_handle(st)
    m = c_double()
    bx = c_double()
    by = c_double()
    bk = c_int32()
    g = lib().ref_graspable(h.ptr, 0, ctypes.byref(params), ctypes.byref(m), ctypes.byref(bx),
                            ctypes.byref(by), ctypes.byref(bk))
    return bool(g), m.value, bx.value, by.value, bk.value


def keyed_picks(seed: int, it: int, env: int, count: int, n: int) -> np.ndarray:
    out = np.zeros(count, np.uint64)
    lib().ref_keyed_picks(seed, it, env, count, n, u64ptr(out))
    return out


def keyed_raw(seed: int, it: int, env: int, count: int) -> np.ndarray:
    out = np.zeros(count, np.uint64)
    lib().ref_keyed_raw(seed, it, env, count, u64ptr(out))
    return out


def mix_keys(seed: int, a: int, b: int = 0) -> int:
    return int(lib().ref_mix_keys(seed, a, b))


def episode_seed(base: int, case_id: str, trial: int) -> int:
    return int(lib().ref_episode_seed(base, case_id.encode(), trial))


def run_search(st: WorldState, params: PpgParams, threads: int = 1, serial: bool = False,
               want_sig: bool = False):
    """run_pmbs (pmbs.cpp:242-292) / run_serial_mcts (mcts.cpp:237-282)."""
    h = state_handle(st)
    action = np.zeros(4, np.float64)
    stats = PpgSearchStats()
    slen = c_int64()
    L = lib()
    rc = L.ref_run_search(h.ptr, 0, ctypes.byref(params), threads, 1 if serial else 0, dptr(action),
                          ctypes.byref(stats), None, 0, ctypes.byref(slen))
    if rc != 0:
        return {"rc": rc}
    sig = None
    if want_sig:
        buf = ctypes.create_string_buffer(slen.value + 1)
        L.ref_run_search(h.ptr, 0, ctypes.byref(params), threads, 1 if serial else 0, dptr(action),
                         ctypes.byref(stats), buf, slen.value + 1, ctypes.byref(slen))
        sig = buf.value.decode()
    return {"rc": 0, "action": action, "iterations": stats.iterations, "expansions": stats.expansions,
            "elapsed_s": stats.elapsed_s, "stop": STOP_REASONS[stats.stop_reason],
            "final_tree_depth": stats.final_tree_depth, "sig_fnv": int(stats.signature_fnv),
            "n_nodes": stats.n_nodes, "sig": sig}


def first_iteration(st: WorldState, params: PpgParams, iteration: int = 0):
    h = state_handle(st)
    N = params.n_envs
    poses = np.zeros((N, st.n, 3), np.float64)
    meta = np.zeros((N, 3), np.int32)
    rewards = np.zeros(N, np.float64)
    cap = c_int32()
    k = lib().ref_first_iteration(h.ptr, 0, ctypes.byref(params), iteration, dptr(poses), iptr(meta),
                                  dptr(rewards), ctypes.byref(cap))
    if k < 0:
        raise RuntimeError("no legal push at the root")
    return poses[:k].copy(), meta[:k].copy(), rewards[:k].copy(), cap.value


def run_episode(st: WorldState, case_id: str, trial: int, params: PpgParams, threads: int = 1,
                seed_base: int = 0, action_cap: int = 16, log_path: str = ""):
    """bench::run_episode (bench.cpp:54-126), optionally writing its JSONL log."""
    h = state_handle(st)
    comp = c_int32()
    ps = c_double()
    used = lib().ref_run_episode(h.ptr, 0, case_id.encode(), trial, ctypes.byref(params), threads,
                                 seed_base, action_cap, ctypes.byref(comp), ctypes.byref(ps), log_path.encode())
    return {"actions_used": used, "completed": bool(comp.value), "planning_s": ps.value}


def replay_log(path: str):
    """bench::replay_log (bench.cpp:319-377): (ok, report)."""
    buf = ctypes.create_string_buffer(4096)
    ok = lib().ref_replay_log(path.encode(), buf, 4096)
    return bool(ok), buf.value.decode()


def c3_trees(variant: int, count: int = 200, cap_nodes: int = 200000, cap_pairs: int = 200000) -> dict:
    """Acceptance criterion 3 (acceptance.cpp:255-281) on the reference:
    random explicit trees + the reference select_batch (ref_shim.cpp
    ref_c3_trees).  Flat per-node / per-pair arrays with offsets."""
    a = {"node_off": np.zeros(count + 1, np.int32), "parent": np.zeros(cap_nodes, np.int32),
         "depth": np.zeros(cap_nodes, np.int32), "visits": np.zeros(cap_nodes, np.int64),
         "q_sum": np.zeros(cap_nodes, np.float64), "flags": np.zeros(cap_nodes, np.uint8),
         "n_children": np.zeros(cap_nodes, np.int32), "n_untried": np.zeros(cap_nodes, np.int32),
         "vv": np.zeros(cap_nodes, np.int64), "pair_off": np.zeros(count + 1, np.int32),
         "sel_node": np.zeros(cap_pairs, np.int32), "sel_untried": np.zeros(cap_pairs, np.int32),
         "tree_depth": np.zeros(count, np.int32), "n_envs": np.zeros(count, np.int32),
         "vsum": np.zeros(count, np.int64), "exhausted": np.zeros(count, np.int32)}
    keys = ["node_off", "parent", "depth", "visits", "q_sum", "flags", "n_children", "n_untried", "vv", "pair_off",
            "sel_node", "sel_untried", "tree_depth", "n_envs", "vsum", "exhausted"]
    rc = lib().ref_c3_trees(variant, count, cap_nodes, cap_pairs, *[a[k].ctypes.data for k in keys])
    if rc != 0:
        raise RuntimeError(f"ref_c3_trees: capacity ({rc})")
    nn, npairs = int(a["node_off"][-1]), int(a["pair_off"][-1])
    for k in ("parent", "depth", "visits", "q_sum", "flags", "n_children", "n_untried", "vv"):
        a[k] = a[k][:nn].copy()
    for k in ("sel_node", "sel_untried"):
        a[k] = a[k][:npairs].copy()
    return a


def batch_simulate(states, node_meta: np.ndarray, params: PpgParams, iteration: int, depth_cap: int,
                   threads: int = 1):
    """pmbs::batch_simulate (pmbs.cpp:207-234) on explicit nodes (one
    WorldState per node, node_meta [n][3] = depth, graspable, dead).  Returns
    (rewards, seconds of the reference call)."""
    from paper_2207_06649_b200.world import ShapeTable as _ST
    node_meta = np.ascontiguousarray(node_meta, np.int32)
    n = len(node_meta)
    h = states_handle(_ST.per_env(list(states)), np.stack([s.poses for s in states]))
    rew = np.zeros(n, np.float64)
    secs = c_double()
    rc = lib().ref_batch_simulate(h.ptr, iptr(node_meta), n, ctypes.byref(params), iteration, depth_cap, threads,
                                  dptr(rew), ctypes.byref(secs))
    if rc != 0:
        raise RuntimeError("ref_batch_simulate failed")
    return rew, secs.value
