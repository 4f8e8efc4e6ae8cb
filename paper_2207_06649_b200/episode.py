"""Object-retrieval episodes on the GPU planner: the caller of
the hot path, restating bench::run_episode (bench.cpp:54-126) and
episode_seed (bench.cpp:50-52) over this package's device API.

Each step: graspable(live) on the device -> grasp and stop, or plan one push
with run_pmbs (step seed mix_keys(seed, step)) and execute it with
resolve_push (a SimError executes as a no-op), capped at `action_cap`
actions.  The optional JSONL log has the reference's records (init / push
with pre/post state digests / grasp), so the reference's own replay_log
(bench.cpp:319-377) can verify it.
"""
from __future__ import annotations

import json
import time
from dataclasses import dataclass, replace
from typing import Optional, TextIO

import numpy as np

from . import abi
from .api import Context, ParallelConfig, SearchError, SimError, default_context, graspable, resolve_push, run_pmbs
from .world import ShapeTable, WorldState

M64 = 0xFFFFFFFFFFFFFFFF


def splitmix64(x: int) -> int:  # rng.hpp:8-13
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def mix_keys(seed: int, a: int, b: int = 0) -> int:  # rng.hpp:15-17
    return splitmix64(splitmix64(splitmix64(seed & M64) ^ (a & M64)) ^ (b & M64))


def fnv1a(s: str) -> int:  # bench.cpp:20-27
    h = 1469598103934665603
    for c in s.encode():
        h ^= c
        h = (h * 1099511628211) & M64
    return h


def episode_seed(seed_base: int, case_id: str, trial: int) -> int:  # bench.cpp:50-52
    return (seed_base + mix_keys(fnv1a(case_id), trial)) & M64


@dataclass
class EpisodeResult:  # bench.hpp:16-26
    case_id: str
    trial: int
    planner: str = "pmbs"
    actions_used: int = 0
    planning_time_s: float = 0.0
    completed: bool = False
    grasp_success: bool = False
    grasp_attempted: bool = False
    threshold_marginal: bool = False
    decisions: int = 0
    env_steps: int = 0


def state_digest(st: WorldState) -> int:
    lib = abi.load_library()
    t = ShapeTable.shared(st)
    out = np.zeros(1, np.uint64)
    poses = np.ascontiguousarray(st.poses.reshape(1, st.n, 3))
    lib.ppg_state_digest(t.struct(), abi.dptr(poses), 1, abi.u64ptr(out))
    return int(out[0])


def scene_json(st: WorldState) -> dict:
    """scene_to_json (world.cpp:230-253)."""
    objs = []
    for i in range(st.n):
        pose = [float(v) for v in st.poses[i]]
        if st.kind[i] == abi.PPG_DISC:
            objs.append({"kind": "disc", "pose": pose, "radius": float(st.radius[i])})
        else:
            vs = [[float(st.vertices[i, k, 0]), float(st.vertices[i, k, 1])] for k in range(st.n_vertices[i])]
            objs.append({"kind": "polygon", "pose": pose, "vertices": vs})
    ws = {"side_length": float(st.side_length)}
    if st.boundary_margin != 0.0:
        ws["boundary_margin"] = float(st.boundary_margin)
    return {"objects": objs, "target_index": int(st.target_index), "workspace": ws}


def _dump(rec: dict) -> str:
    return json.dumps(rec, sort_keys=True, separators=(",", ":"))


def run_episode(scene: WorldState, case_id: str, trial: int, cfg: ParallelConfig, seed: int,
                action_cap: int = 16, log: Optional[TextIO] = None, ctx: Optional[Context] = None) -> EpisodeResult:
    ctx = ctx or default_context()
    res = EpisodeResult(case_id, trial)
    live = scene.copy()
    if log is not None:
        log.write(_dump({"type": "init", "case_id": case_id, "trial": trial, "planner": "pmbs",
                         "sim": {"push_distance": cfg.sim.push_distance, "substeps": cfg.sim.substeps,
                                 "max_projection_iters": cfg.sim.max_projection_iters, "eps_pen": cfg.sim.eps_pen,
                                 "rotation_gain": cfg.sim.rotation_gain, "tip": [cfg.tip.radius, cfg.tip.clearance]},
                         "state": scene_json(scene)}) + "\n")
    step = 0
    while res.actions_used < action_cap:
        report = graspable(live, cfg.grasp, cfg.margin_threshold, ctx=ctx)
        if not report.graspable and report.best is not None:
            res.threshold_marginal = True
        if report.graspable:
            res.grasp_attempted = True
            res.actions_used += 1
            pose = report.best  # best_grasp == graspable(state, geom, 0.0).best (actions.cpp:149-151)
            res.grasp_success = pose is not None
            res.completed = res.grasp_success
            if log is not None:
                rec = {"type": "grasp", "success": res.grasp_success}
                if pose is not None:
                    rec.update({"x": pose[0], "y": pose[1], "angle_index": pose[2]})
                log.write(_dump(rec) + "\n")
            break
        step_cfg = replace(cfg, rng_seed=mix_keys(seed, step))
        t0 = time.perf_counter()
        try:
            plan = run_pmbs(live, step_cfg, ctx=ctx)
        except SearchError:
            break  # no legal pushes: incomplete episode
        res.planning_time_s += time.perf_counter() - t0
        res.decisions += 1
        res.env_steps += plan.env_steps
        pre = state_digest(live)
        applied = True
        try:
            live = resolve_push(live, plan.action, cfg.tip, cfg.sim, ctx=ctx)
        except SimError:
            applied = False  # a jammed push executes as a no-op
        res.actions_used += 1
        step += 1
        if log is not None:
            log.write(_dump({"type": "push", "action": [float(v) for v in plan.action], "applied": applied,
                             "pre": str(pre), "post": str(state_digest(live))}) + "\n")
    return res
