"""Host-side scene types mirroring the reference world model.

``WorldState`` mirrors pushplan::WorldState (world.hpp:62-71): shapes
(ObjectShape world.hpp:33-46), poses (Pose world.hpp:49-56), target index and
workspace (world.hpp:17-30).  ``ShapeTable`` packs one or many states into the
flat arrays of the C-ABI (include/pushplan_gpu.h ``ppg_shapes``).
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from typing import List, Sequence

import numpy as np

from .abi import PPG_DISC, PPG_MAX_OBJECTS, PPG_MAX_VERTICES, PPG_POLYGON, PpgShapes, dptr, iptr


class SceneError(ValueError):
    """Reference SceneError (world.hpp:12)."""


def wrap_angle(theta: float) -> float:
    """geometry.cpp:8-13 — math.fmod is C fmod (exact), so this is bit-identical."""
    two_pi = 2.0 * math.pi
    t = math.fmod(theta + math.pi, two_pi)
    if t < 0.0:
        t += two_pi
    return t - math.pi


@dataclass
class WorldState:
    kind: np.ndarray                 # int32 [n]
    radius: np.ndarray               # f64 [n] (0.0 for polygons, as ObjectShape::polygon leaves it)
    n_vertices: np.ndarray           # int32 [n]
    vertices: np.ndarray             # f64 [n, PPG_MAX_VERTICES, 2]
    poses: np.ndarray                # f64 [n, 3]
    target_index: int = 0
    side_length: float = 0.288
    boundary_margin: float = 0.0

    @property
    def n(self) -> int:
        return int(self.kind.shape[0])

    @property
    def all_discs(self) -> bool:
        return bool(np.all(self.kind == PPG_DISC))

    def copy(self) -> "WorldState":
        return WorldState(self.kind.copy(), self.radius.copy(), self.n_vertices.copy(),
                          self.vertices.copy(), self.poses.copy(), self.target_index,
                          self.side_length, self.boundary_margin)

    def with_poses(self, poses: np.ndarray) -> "WorldState":
        s = self.copy()
        s.poses = np.ascontiguousarray(poses, dtype=np.float64).reshape(self.n, 3)
        return s

    @staticmethod
    def from_objects(objects: Sequence[dict], target_index: int = 0, side_length: float = 0.288,
                     boundary_margin: float = 0.0) -> "WorldState":
        """objects: dicts {kind: 'disc'|'polygon', radius|vertices, pose: [x, y, theta]}."""
        n = len(objects)
        if n == 0:
            raise SceneError("scene has no objects")
        if n > PPG_MAX_OBJECTS:
            raise SceneError(f"at most {PPG_MAX_OBJECTS} objects are supported")
        kind = np.zeros(n, np.int32)
        radius = np.zeros(n, np.float64)
        nv = np.zeros(n, np.int32)
        verts = np.zeros((n, PPG_MAX_VERTICES, 2), np.float64)
        poses = np.zeros((n, 3), np.float64)
        for i, o in enumerate(objects):
            if o["kind"] == "disc":
                kind[i] = PPG_DISC
                radius[i] = float(o["radius"])
            elif o["kind"] == "polygon":
                kind[i] = PPG_POLYGON
                vs = o["vertices"]
                if len(vs) > PPG_MAX_VERTICES:
                    raise SceneError(f"at most {PPG_MAX_VERTICES} polygon vertices are supported")
                nv[i] = len(vs)
                for k, v in enumerate(vs):
                    verts[i, k] = (float(v[0]), float(v[1]))
            else:
                raise SceneError(f"unknown object kind: {o['kind']}")
            p = o["pose"]
            poses[i] = (float(p[0]), float(p[1]), float(p[2]))
        return WorldState(kind, radius, nv, verts, poses, int(target_index), float(side_length),
                          float(boundary_margin))


def scene_from_json_text(text: str) -> WorldState:
    """scene_from_json (world.cpp:197-228): theta is wrapped on load; the
    structural invariants of WorldState::validate (world.cpp:72-84) are checked
    except the penetration bound, which the device checks on first use."""
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as e:
        raise SceneError(f"scene parse error: {e}") from e
    ws = doc.get("workspace", {})
    objs = []
    for o in doc["objects"]:
        p = o["pose"]
        o = dict(o)
        o["pose"] = [p[0], p[1], wrap_angle(float(p[2]))]
        objs.append(o)
    st = WorldState.from_objects(objs, doc["target_index"], ws.get("side_length", 0.288),
                                 ws.get("boundary_margin", 0.0))
    validate(st)
    return st


def load_scene(path: str) -> WorldState:
    """load_scene (world.cpp:271-277)."""
    with open(path) as f:
        return scene_from_json_text(f.read())


def validate(st: WorldState) -> None:
    """Structural part of WorldState::validate (world.cpp:72-84)."""
    if not st.side_length > 0.0:
        raise SceneError("workspace side_length must be > 0")
    if st.boundary_margin < 0.0 or st.boundary_margin >= st.side_length / 2.0:
        raise SceneError("workspace boundary_margin out of range")
    if not 0 <= st.target_index < st.n:
        raise SceneError("target_index out of range")
    if not np.all(np.isfinite(st.poses)):
        raise SceneError("pose values must be finite")
    h = st.side_length / 2.0 - st.boundary_margin
    if not np.all((np.abs(st.poses[:, 0]) < h) & (np.abs(st.poses[:, 1]) < h)):
        raise SceneError("object center outside workspace boundary")
    for i in range(st.n):
        if st.kind[i] == PPG_DISC and not st.radius[i] > 0.0:
            raise SceneError("disc radius must be > 0")
        if st.kind[i] == PPG_POLYGON and st.n_vertices[i] < 3:
            raise SceneError("polygon must be convex, non-degenerate and counter-clockwise")


@dataclass
class ShapeTable:
    """Flat ppg_shapes arrays for a batch: one table (shared) or one per env."""
    kind: np.ndarray
    radius: np.ndarray
    n_vertices: np.ndarray
    vertices: np.ndarray
    target_index: np.ndarray
    side_length: float
    boundary_margin: float
    n_objects: int
    n_tables: int
    _struct: PpgShapes = field(default=None, repr=False)

    @staticmethod
    def shared(st: WorldState) -> "ShapeTable":
        return ShapeTable(np.ascontiguousarray(st.kind, np.int32),
                          np.ascontiguousarray(st.radius, np.float64),
                          np.ascontiguousarray(st.n_vertices, np.int32),
                          np.ascontiguousarray(st.vertices, np.float64),
                          np.array([st.target_index], np.int32), st.side_length,
                          st.boundary_margin, st.n, 1)

    @staticmethod
    def per_env(states: List[WorldState]) -> "ShapeTable":
        n = states[0].n
        for s in states:
            if s.n != n:
                raise ValueError("a batch must have a uniform object count")
            if s.side_length != states[0].side_length or s.boundary_margin != states[0].boundary_margin:
                raise ValueError("a batch must share one workspace")
        return ShapeTable(np.ascontiguousarray(np.stack([s.kind for s in states]), np.int32),
                          np.ascontiguousarray(np.stack([s.radius for s in states]), np.float64),
                          np.ascontiguousarray(np.stack([s.n_vertices for s in states]), np.int32),
                          np.ascontiguousarray(np.stack([s.vertices for s in states]), np.float64),
                          np.array([s.target_index for s in states], np.int32),
                          states[0].side_length, states[0].boundary_margin, n, len(states))

    def struct(self) -> PpgShapes:
        if self._struct is None:
            self._struct = PpgShapes(self.n_objects, self.n_tables, iptr(self.kind), dptr(self.radius),
                                     iptr(self.n_vertices), dptr(self.vertices),
                                     iptr(self.target_index), self.side_length, self.boundary_margin)
        return self._struct


def stack_poses(states: List[WorldState]) -> np.ndarray:
    return np.ascontiguousarray(np.stack([s.poses for s in states]), np.float64)
