"""Reference-shaped Python API over the C-ABI (include/pushplan_gpu.h).

Names, argument meaning and error behaviour follow the reference planner /
simulator interface (/root/reference/proj/core/include/pushplan/*.hpp):

    batch_resolve(states, pushes, tip, params)      push_sim.hpp:48-51
    resolve_push(state, push, tip, params)          push_sim.hpp:34-35 (raises SimError)
    sample_pushes(state, n_per_object, tip, dist)   actions.hpp:39-40
    graspable(state, geom, margin_threshold)        actions.hpp:47-48
    run_pmbs(state, cfg)                            pmbs.hpp:91 (raises SearchError)

Every call runs on the GPU through libpmbs_b200.so; there is no CPU path.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import abi
from .abi import PpgParams, PpgSearchStats, dptr, i64ptr, iptr, u8ptr
from .world import ShapeTable, WorldState, stack_poses


class SimError(RuntimeError):
    """push_sim.hpp:22"""


class SearchError(RuntimeError):
    """mcts.hpp:15"""


class DeviceError(RuntimeError):
    """CUDA failure or no device (the product has no CPU fallback)."""


@dataclass
class GripperTip:  # world.hpp:86-89
    radius: float = 0.012
    clearance: float = 0.002


@dataclass
class SimParams:  # push_sim.hpp:14-20
    push_distance: float = 0.05
    substeps: int = 64
    max_projection_iters: int = 32
    eps_pen: float = 1e-4
    rotation_gain: float = 1.0


@dataclass
class GraspGeometry:  # actions.hpp:21-26
    finger_width: float = 0.02
    finger_thickness: float = 0.01
    opening: float = 0.085
    approach_clearance: float = 0.003


@dataclass
class Budget:  # mcts.hpp:20-28
    mode: str = "seconds"
    max_seconds: float = 60.0
    max_iterations: int = 0

    @staticmethod
    def seconds(s: float) -> "Budget":
        return Budget("seconds", s, 0)

    @staticmethod
    def iterations(n: int) -> "Budget":
        return Budget("iterations", 0.0, n)


@dataclass
class ParallelConfig:  # SearchConfig mcts.hpp:30-44 + ParallelConfig pmbs.hpp:24-28
    gamma: float = 0.8
    c_explore: float = 0.3
    tree_depth: int = 7
    rollout_depth: int = 3
    budget: Budget = field(default_factory=Budget)
    pushes_per_object: int = 16
    margin_threshold: float = 0.003
    rng_seed: int = 0
    rank_by_ucb: bool = False
    tip: GripperTip = field(default_factory=GripperTip)
    grasp: GraspGeometry = field(default_factory=GraspGeometry)
    sim: SimParams = field(default_factory=SimParams)
    n_envs: int = 64
    worker_threads: int = 1  # accepted for API parity; the device replaces the pool
    leaf_parallel: bool = True

    def to_params(self) -> PpgParams:
        return abi.default_params(
            tip_radius=self.tip.radius, tip_clearance=self.tip.clearance,
            push_distance=self.sim.push_distance, substeps=self.sim.substeps,
            max_projection_iters=self.sim.max_projection_iters, eps_pen=self.sim.eps_pen,
            rotation_gain=self.sim.rotation_gain, finger_width=self.grasp.finger_width,
            finger_thickness=self.grasp.finger_thickness, opening=self.grasp.opening,
            approach_clearance=self.grasp.approach_clearance, gamma=self.gamma,
            c_explore=self.c_explore, tree_depth=self.tree_depth, rollout_depth=self.rollout_depth,
            pushes_per_object=self.pushes_per_object, margin_threshold=self.margin_threshold,
            rng_seed=self.rng_seed & 0xFFFFFFFFFFFFFFFF, rank_by_ucb=int(self.rank_by_ucb),
            budget_iterations=int(self.budget.mode == "iterations"),
            max_iterations=self.budget.max_iterations, max_seconds=self.budget.max_seconds,
            n_envs=self.n_envs, leaf_parallel=int(self.leaf_parallel))


@dataclass
class PushResult:  # push_sim.hpp:38-43
    state: Optional[WorldState]
    error: str = ""

    def ok(self) -> bool:
        return self.state is not None


@dataclass
class GraspReport:  # actions.hpp:28-32
    graspable: bool
    margin: float
    best: Optional[tuple]  # (x, y, angle_index)


@dataclass
class SearchResult:  # mcts.hpp:80-91
    action: np.ndarray
    iterations: int
    expansions: int
    elapsed_s: float
    stop_reason: str
    final_tree_depth: int
    env_steps: int
    rollout_steps: int
    lockstep_rounds: int
    signature_fnv: int
    n_nodes: int
    signature: Optional[str] = None
    phase_s: Optional[dict] = None


_ERRS = {abi.PPG_EINVAL: "invalid argument", abi.PPG_ECUDA: "CUDA error",
         abi.PPG_ENOLEGAL: "no legal push action at the root", abi.PPG_ENODEVICE: "no CUDA device"}


class Context:
    """One device context (the reference WorkerPool seam).  Not thread-safe:
    one context per host thread, as the C-ABI states."""

    def __init__(self, device: int = 0, params: Optional[PpgParams] = None, _create=None):
        self.lib = abi.load_library()
        err = ctypes.c_int()
        self.params = params if params is not None else abi.default_params()
        if _create is None:
            self.ptr = self.lib.ppg_create(device, ctypes.byref(self.params), ctypes.byref(err))
        else:
            self.ptr = _create(self.lib, self.params, err)
        if not self.ptr:
            raise DeviceError(f"context creation failed: {_ERRS.get(err.value, err.value)}")
        self.device = device
        self._scene_key = None

    # ---- multi-GPU contexts (csrc/multi.cu) ----------------------
    @classmethod
    def multi(cls, devices: Sequence[int], params: Optional[PpgParams] = None, emulate: bool = False) -> "Context":
        """One process driving several GPUs (ncclCommInitAll): batch_simulate
        and run_pmbs shard the rollout batch over `devices`.  emulate=True:
        the shards all live on one device and exchange through a device
        kernel (the single-GPU test double of the NCCL path)."""
        devs = (ctypes.c_int * len(devices))(*devices)
        flags = abi.PPG_MULTI_EMULATE if emulate else 0
        return cls(devices[0], params, lambda lib, p, err: lib.ppg_create_multi(devs, len(devices), flags,
                                                                              ctypes.byref(p), ctypes.byref(err)))

    @classmethod
    def rank(cls, device: int, rank: int, world: int, nccl_id: Optional[bytes],
             params: Optional[PpgParams] = None) -> "Context":
        """One shard per process (torchrun): rank `rank` of `world`, NCCL
        communicator from the 128-byte id rank 0 made (nccl_unique_id)."""
        buf = ctypes.create_string_buffer(bytes(nccl_id), 128) if nccl_id is not None else None
        return cls(device, params, lambda lib, p, err: lib.ppg_create_rank(device, rank, world, buf, ctypes.byref(p),
                                                                         ctypes.byref(err)))

    def shard_info(self) -> dict:
        r, w, h, t = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        self._check(self.lib.ppg_shard_info(self.ptr, ctypes.byref(r), ctypes.byref(w), ctypes.byref(h),
                                            ctypes.byref(t)), "ppg_shard_info")
        return {"rank": r.value, "world": w.value, "shards_here": h.value,
                "transport": {0: "none", 1: "nccl", 2: "emulated"}[t.value]}

    def close(self):
        if getattr(self, "ptr", None):
            self.lib.ppg_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        self.close()

    def _check(self, rc: int, what: str):
        if rc == abi.PPG_SUCCESS:
            return
        msg = self.lib.ppg_last_error(self.ptr).decode()
        if rc == abi.PPG_ENOLEGAL:
            raise SearchError(msg or "no legal push action at the root")
        if rc == abi.PPG_EINVAL:
            raise ValueError(f"{what}: {msg}")
        raise DeviceError(f"{what}: {msg}")

    def set_planner(self, mode: str):
        """"auto" (device tree unless a simulate hook is installed), "host"
        (planner.cpp) or "device" (dtree.cu) for run_pmbs."""
        code = {"auto": abi.PPG_PLANNER_AUTO, "host": abi.PPG_PLANNER_HOST, "device": abi.PPG_PLANNER_DEVICE}[mode]
        self._check(self.lib.ppg_set_planner(self.ptr, code), "ppg_set_planner")

    def set_params(self, params: PpgParams):
        self.params = params
        self._check(self.lib.ppg_set_params(self.ptr, ctypes.byref(params)), "ppg_set_params")

    def set_scene(self, st: WorldState):
        key = (st.kind.tobytes(), st.radius.tobytes(), st.n_vertices.tobytes(), st.vertices.tobytes(),
               st.target_index, st.side_length, st.boundary_margin)
        if key == self._scene_key:
            return
        self._scene_table = ShapeTable.shared(st)
        self._check(self.lib.ppg_set_scene(self.ptr, ctypes.byref(self._scene_table.struct())), "ppg_set_scene")
        self._scene_key = key

    # ---- batched primitives -------------------------------------------------
    def batch_resolve_arrays(self, table: Optional[ShapeTable], poses: np.ndarray, pushes: np.ndarray, out=None):
        """`out` = optional caller-owned (poses_out, status, residual) arrays;
        pinned host buffers (e.g. numpy views of pinned torch tensors) let the
        kernel write results directly (zero-copy output)."""
        poses = np.ascontiguousarray(poses, np.float64)
        pushes = np.ascontiguousarray(pushes, np.float64)
        E = poses.shape[0]
        if pushes.shape[0] != E:
            raise SimError("batch_resolve: states and pushes must have equal length")
        if out is not None:
            out, status, resid = out
            if (out.shape != poses.shape or out.dtype != np.float64 or not out.flags.c_contiguous or
                    status.shape != (E,) or status.dtype != np.int32 or resid.shape != (E,) or
                    resid.dtype != np.float64):
                raise ValueError("batch_resolve_arrays: out arrays must match the batch (f64 poses, i32, f64)")
        else:
            out = np.empty_like(poses)
            status = np.empty(E, np.int32)
            resid = np.empty(E, np.float64)
        sh = ctypes.byref(table.struct()) if table is not None else None
        self._check(self.lib.ppg_batch_resolve(self.ptr, sh, dptr(poses), dptr(pushes), E, dptr(out), iptr(status),
                                               dptr(resid)), "ppg_batch_resolve")
        return out, status, resid

    def sample_pushes_arrays(self, poses: np.ndarray, table: Optional[ShapeTable] = None):
        poses = np.ascontiguousarray(poses, np.float64)
        E, n = poses.shape[0], poses.shape[1]
        cap = n * self.params.pushes_per_object
        out = np.empty((E, cap, 4), np.float64)
        cnt = np.empty(E, np.int32)
        sh = ctypes.byref(table.struct()) if table is not None else None
        self._check(self.lib.ppg_sample_pushes(self.ptr, sh, dptr(poses), E, dptr(out), iptr(cnt)),
                    "ppg_sample_pushes")
        return out, cnt

    def graspable_arrays(self, poses: np.ndarray):
        poses = np.ascontiguousarray(poses, np.float64)
        E = poses.shape[0]
        g = np.empty(E, np.uint8)
        m = np.empty(E, np.float64)
        bx = np.empty(E, np.float64)
        by = np.empty(E, np.float64)
        bk = np.empty(E, np.int32)
        self._check(self.lib.ppg_graspable(self.ptr, dptr(poses), E, u8ptr(g), dptr(m), dptr(bx), dptr(by),
                                           iptr(bk)), "ppg_graspable")
        return g, m, bx, by, bk

    def expand_arrays(self, parent_poses: np.ndarray, actions: np.ndarray):
        parent_poses = np.ascontiguousarray(parent_poses, np.float64)
        actions = np.ascontiguousarray(actions, np.float64)
        P, n = parent_poses.shape[0], parent_poses.shape[1]
        cap = n * self.params.pushes_per_object
        child = np.empty_like(parent_poses)
        status = np.empty(P, np.int32)
        g = np.empty(P, np.uint8)
        nu = np.empty(P, np.int32)
        un = np.empty((P, cap, 4), np.float64)
        self._check(self.lib.ppg_expand(self.ptr, dptr(parent_poses), dptr(actions), P, dptr(child), iptr(status),
                                        u8ptr(g), iptr(nu), dptr(un)), "ppg_expand")
        return child, status, g, nu, un

    def simulate_arrays(self, node_poses: np.ndarray, node_meta: np.ndarray, n_envs: int, leaf_parallel: bool,
                        seed: int, iteration: int, depth_cap: int):
        node_poses = np.ascontiguousarray(node_poses, np.float64)
        node_meta = np.ascontiguousarray(node_meta, np.int32)
        nn = node_poses.shape[0]
        rewards = np.zeros(nn, np.float64)
        ctr = np.zeros(4, np.int64)
        self._check(self.lib.ppg_simulate(self.ptr, dptr(node_poses), iptr(node_meta), nn, n_envs,
                                          int(leaf_parallel), seed & 0xFFFFFFFFFFFFFFFF, iteration, depth_cap,
                                          dptr(rewards), i64ptr(ctr)), "ppg_simulate")
        return rewards, ctr

    def simulate_count_arrays(self, node_poses: np.ndarray, node_meta: np.ndarray, n_envs: int,
                              leaf_parallel: bool, seed: int, iteration: int, depth_cap: int):
        """The algorithmic FP64 work of a simulate_arrays call (same rollouts):
        (ops[3] = resolve, sample, grasp, counters[4])."""
        node_poses = np.ascontiguousarray(node_poses, np.float64)
        node_meta = np.ascontiguousarray(node_meta, np.int32)
        ops = np.zeros(3, np.int64)
        ctr = np.zeros(4, np.int64)
        self._check(self.lib.ppg_simulate_count(self.ptr, dptr(node_poses), iptr(node_meta), node_poses.shape[0],
                                                n_envs, int(leaf_parallel), seed & 0xFFFFFFFFFFFFFFFF, iteration,
                                                depth_cap, i64ptr(ops), i64ptr(ctr)), "ppg_simulate_count")
        return ops, ctr

    def run_pmbs_arrays(self, root_poses: np.ndarray, want_sig: bool = False) -> SearchResult:
        root_poses = np.ascontiguousarray(root_poses, np.float64)
        action = np.zeros(4, np.float64)
        st = PpgSearchStats()
        sig = None
        if want_sig:
            ln = ctypes.c_int64()
            rc = self.lib.ppg_run_pmbs_sig(self.ptr, dptr(root_poses), dptr(action), ctypes.byref(st), None, 0,
                                           ctypes.byref(ln))
            self._check(rc, "ppg_run_pmbs")
            buf = ctypes.create_string_buffer(ln.value + 1)
            rc = self.lib.ppg_run_pmbs_sig(self.ptr, dptr(root_poses), dptr(action), ctypes.byref(st), buf,
                                           ln.value + 1, ctypes.byref(ln))
            self._check(rc, "ppg_run_pmbs")
            sig = buf.value.decode()
        else:
            self._check(self.lib.ppg_run_pmbs(self.ptr, dptr(root_poses), dptr(action), ctypes.byref(st)),
                        "ppg_run_pmbs")
        return SearchResult(action, st.iterations, st.expansions, st.elapsed_s, abi.STOP_REASONS[st.stop_reason],
                            st.final_tree_depth, st.env_steps, st.rollout_steps, st.lockstep_rounds,
                            int(st.signature_fnv), st.n_nodes, sig,
                            {"select": st.select_s, "expand": st.expand_s, "simulate": st.simulate_s,
                             "backprop": st.backprop_s})


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId through the library (rank 0 makes it, the caller
    broadcasts the 128 bytes)."""
    lib = abi.load_library()
    buf = ctypes.create_string_buffer(128)
    if lib.ppg_nccl_unique_id(buf) != abi.PPG_SUCCESS:
        raise DeviceError("ppg_nccl_unique_id: NCCL unavailable")
    return buf.raw


_DEFAULT_CTX: Optional[Context] = None


def default_context() -> Context:
    global _DEFAULT_CTX
    if _DEFAULT_CTX is None:
        _DEFAULT_CTX = Context(0)
    return _DEFAULT_CTX


def _with_params(ctx: Context, tip: GripperTip, params: SimParams, **extra) -> None:
    p = ParallelConfig(tip=tip, sim=params).to_params()
    for k, v in extra.items():
        setattr(p, k, v)
    ctx.set_params(p)


def batch_resolve(states: Sequence[WorldState], pushes: Sequence, tip: GripperTip = GripperTip(),
                  params: SimParams = SimParams(), ctx: Optional[Context] = None) -> List[PushResult]:
    """push_sim.cpp:132-152 — element-wise resolve_push with per-element
    errors; raises SimError on a length mismatch."""
    if len(states) != len(pushes):
        raise SimError("batch_resolve: states and pushes must have equal length")
    if len(states) == 0:
        return []
    ctx = ctx or default_context()
    _with_params(ctx, tip, params)
    results: List[Optional[PushResult]] = [None] * len(states)
    groups = {}
    for i, s in enumerate(states):  # one launch per (object count, workspace)
        groups.setdefault((s.n, s.side_length, s.boundary_margin), []).append(i)
    for idx in groups.values():
        sub = [states[i] for i in idx]
        table = ShapeTable.per_env(sub)
        out, status, resid = ctx.batch_resolve_arrays(table, stack_poses(sub),
                                                      np.asarray([pushes[i] for i in idx], np.float64))
        for k, i in enumerate(idx):
            if status[k] == abi.PPG_OK:
                results[i] = PushResult(states[i].with_poses(out[k]))
            elif status[k] == abi.PPG_START_COLLISION:
                results[i] = PushResult(None, "resolve_push: gripper start pose collides or leaves the workspace")
            else:
                results[i] = PushResult(None, "resolve_push: projection did not converge, residual penetration "
                                              f"{resid[k]:g} m")
    return results


def resolve_push(state: WorldState, push, tip: GripperTip = GripperTip(), params: SimParams = SimParams(),
                 ctx: Optional[Context] = None) -> WorldState:
    r = batch_resolve([state], [push], tip, params, ctx)[0]
    if not r.ok():
        raise SimError(r.error)
    return r.state


def sample_pushes(state: WorldState, n_per_object: int, tip: GripperTip = GripperTip(),
                  push_distance: float = 0.05, ctx: Optional[Context] = None) -> np.ndarray:
    if n_per_object < 1:
        return np.zeros((0, 4), np.float64)
    ctx = ctx or default_context()
    _with_params(ctx, tip, SimParams(push_distance=push_distance), pushes_per_object=n_per_object)
    ctx.set_scene(state)
    out, cnt = ctx.sample_pushes_arrays(state.poses.reshape(1, state.n, 3))
    return out[0, :cnt[0]].copy()


def graspable(state: WorldState, geom: GraspGeometry = GraspGeometry(), margin_threshold: float = 0.003,
              ctx: Optional[Context] = None) -> GraspReport:
    ctx = ctx or default_context()
    p = ParallelConfig(grasp=geom, margin_threshold=margin_threshold).to_params()
    ctx.set_params(p)
    ctx.set_scene(state)
    g, m, bx, by, bk = ctx.graspable_arrays(state.poses.reshape(1, state.n, 3))
    best = (float(bx[0]), float(by[0]), int(bk[0])) if bk[0] >= 0 else None
    return GraspReport(bool(g[0]), float(m[0]), best)


def run_pmbs(state: WorldState, cfg: ParallelConfig = ParallelConfig(), ctx: Optional[Context] = None,
             want_signature: bool = False) -> SearchResult:
    """pmbs.cpp:242-292: one PMBS planning decision on the GPU."""
    ctx = ctx or default_context()
    ctx.set_params(cfg.to_params())
    ctx.set_scene(state)
    return ctx.run_pmbs_arrays(state.poses, want_signature)
