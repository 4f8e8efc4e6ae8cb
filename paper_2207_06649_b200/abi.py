"""ctypes mirror of include/pushplan_gpu.h (the product C-ABI).

The shared library ``libpmbs_b200.so`` is built in-tree (``__graft_entry__.build``)
and loaded from this package directory.  There is no CPU fallback: when the
library or a CUDA device is missing, the calls raise.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_int32, c_int64, c_uint8, c_uint64, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# PPG_LIB: load another build of the library (A/B experiments); default in-tree
LIB_PATH = os.environ.get("PPG_LIB") or os.path.join(HERE, "libpmbs_b200.so")

PPG_MAX_OBJECTS = 32
PPG_MAX_VERTICES = 8

PPG_SUCCESS = 0
PPG_MULTI_EMULATE = 1
PPG_PLANNER_AUTO, PPG_PLANNER_HOST, PPG_PLANNER_DEVICE = 0, 1, 2
PPG_EINVAL = -1
PPG_ECUDA = -2
PPG_ENOLEGAL = -3
PPG_ENODEVICE = -4

PPG_OK = 0
PPG_START_COLLISION = 1
PPG_NOT_CONVERGED = 2

PPG_DISC = 0
PPG_POLYGON = 1

STOP_REASONS = {0: "budget", 1: "explored", 2: "early_stop"}


class PpgShapes(ctypes.Structure):
    _fields_ = [
        ("n_objects", c_int32),
        ("n_tables", c_int32),
        ("kind", POINTER(c_int32)),
        ("radius", POINTER(c_double)),
        ("n_vertices", POINTER(c_int32)),
        ("vertices", POINTER(c_double)),
        ("target_index", POINTER(c_int32)),
        ("side_length", c_double),
        ("boundary_margin", c_double),
    ]


class PpgParams(ctypes.Structure):
    _fields_ = [
        ("tip_radius", c_double),
        ("tip_clearance", c_double),
        ("push_distance", c_double),
        ("substeps", c_int32),
        ("max_projection_iters", c_int32),
        ("eps_pen", c_double),
        ("rotation_gain", c_double),
        ("finger_width", c_double),
        ("finger_thickness", c_double),
        ("opening", c_double),
        ("approach_clearance", c_double),
        ("gamma", c_double),
        ("c_explore", c_double),
        ("tree_depth", c_int32),
        ("rollout_depth", c_int32),
        ("pushes_per_object", c_int32),
        ("margin_threshold", c_double),
        ("rng_seed", c_uint64),
        ("rank_by_ucb", c_int32),
        ("budget_iterations", c_int32),
        ("max_iterations", c_int64),
        ("max_seconds", c_double),
        ("n_envs", c_int32),
        ("leaf_parallel", c_int32),
    ]


class PpgSearchStats(ctypes.Structure):
    _fields_ = [
        ("iterations", c_int64),
        ("expansions", c_int64),
        ("elapsed_s", c_double),
        ("stop_reason", c_int32),
        ("final_tree_depth", c_int32),
        ("env_steps", c_int64),
        ("rollout_steps", c_int64),
        ("lockstep_rounds", c_int64),
        ("signature_fnv", c_uint64),
        ("n_nodes", c_int64),
        ("select_s", c_double),
        ("expand_s", c_double),
        ("simulate_s", c_double),
        ("backprop_s", c_double),
    ]


def default_params(**overrides) -> PpgParams:
    """Reference defaults (GripperTip, SimParams, GraspGeometry, SearchConfig,
    ParallelConfig: world.hpp:86-89, push_sim.hpp:14-20, actions.hpp:21-26,
    mcts.hpp:30-44, pmbs.hpp:24-28)."""
    p = PpgParams(
        tip_radius=0.012, tip_clearance=0.002, push_distance=0.05, substeps=64,
        max_projection_iters=32, eps_pen=1e-4, rotation_gain=1.0, finger_width=0.02,
        finger_thickness=0.01, opening=0.085, approach_clearance=0.003, gamma=0.8,
        c_explore=0.3, tree_depth=7, rollout_depth=3, pushes_per_object=16,
        margin_threshold=0.003, rng_seed=0, rank_by_ucb=0, budget_iterations=0,
        max_iterations=0, max_seconds=60.0, n_envs=64, leaf_parallel=1)
    for k, v in overrides.items():
        setattr(p, k, v)
    return p


def dptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(POINTER(c_double))


def iptr(a: np.ndarray):
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(POINTER(c_int32))


def i64ptr(a: np.ndarray):
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(POINTER(c_int64))


def u64ptr(a: np.ndarray):
    assert a.dtype == np.uint64 and a.flags.c_contiguous
    return a.ctypes.data_as(POINTER(c_uint64))


def u8ptr(a: np.ndarray):
    assert a.dtype == np.uint8 and a.flags.c_contiguous
    return a.ctypes.data_as(POINTER(c_uint8))


# Every symbol include/pushplan_gpu.h declares, with its ctypes signature.
SIGNATURES = {
    "ppg_params_default": (None, [POINTER(PpgParams)]),
    "ppg_version": (c_char_p, []),
    "ppg_device_count": (c_int, []),
    "ppg_create": (c_void_p, [c_int, POINTER(PpgParams), POINTER(c_int)]),
    "ppg_destroy": (None, [c_void_p]),
    "ppg_last_error": (c_char_p, [c_void_p]),
    "ppg_set_params": (c_int, [c_void_p, POINTER(PpgParams)]),
    "ppg_set_scene": (c_int, [c_void_p, POINTER(PpgShapes)]),
    "ppg_batch_resolve": (c_int, [c_void_p, POINTER(PpgShapes), POINTER(c_double), POINTER(c_double),
                                  c_int, POINTER(c_double), POINTER(c_int32), POINTER(c_double)]),
    "ppg_batch_resolve_dev": (c_int, [c_void_p, POINTER(PpgShapes), c_void_p, c_void_p, c_int,
                                      c_void_p, c_void_p, c_void_p, c_void_p]),
    "ppg_sample_pushes": (c_int, [c_void_p, POINTER(PpgShapes), POINTER(c_double), c_int, POINTER(c_double),
                                  POINTER(c_int32)]),
    "ppg_graspable": (c_int, [c_void_p, POINTER(c_double), c_int, POINTER(c_uint8), POINTER(c_double),
                              POINTER(c_double), POINTER(c_double), POINTER(c_int32)]),
    "ppg_expand": (c_int, [c_void_p, POINTER(c_double), POINTER(c_double), c_int, POINTER(c_double),
                           POINTER(c_int32), POINTER(c_uint8), POINTER(c_int32), POINTER(c_double)]),
    "ppg_simulate": (c_int, [c_void_p, POINTER(c_double), POINTER(c_int32), c_int, c_int, c_int,
                             c_uint64, c_uint64, c_int, POINTER(c_double), POINTER(c_int64)]),
    "ppg_run_pmbs": (c_int, [c_void_p, POINTER(c_double), POINTER(c_double), POINTER(PpgSearchStats)]),
    "ppg_run_pmbs_sig": (c_int, [c_void_p, POINTER(c_double), POINTER(c_double),
                                 POINTER(PpgSearchStats), c_char_p, c_int64, POINTER(c_int64)]),
    "ppg_state_digest": (c_int, [POINTER(PpgShapes), POINTER(c_double), c_int, POINTER(c_uint64)]),
    "ppg_batch_resolve_count_dev": (c_int, [c_void_p, POINTER(PpgShapes), c_void_p, c_void_p, c_int,
                                            c_void_p, c_void_p]),
    "ppg_lock_begin": (c_int, [c_void_p, POINTER(c_double), POINTER(c_int32), c_int, c_int, c_int, c_int, c_int,
                               c_uint64, c_uint64, c_int]),
    "ppg_lock_report": (c_int, [c_void_p, POINTER(c_int32), POINTER(c_int32), POINTER(c_uint8), POINTER(c_double),
                                POINTER(c_int32), POINTER(c_int32), POINTER(c_int32)]),
    "ppg_lock_repurpose": (c_int, [c_void_p, POINTER(c_int32), POINTER(c_int32), c_int]),
    "ppg_lock_step": (c_int, [c_void_p]),
    "ppg_lock_counters": (c_int, [c_void_p, POINTER(c_int64)]),
    "ppg_set_simulate_hook": (c_int, [c_void_p, c_void_p, c_void_p]),
    "ppg_set_planner": (c_int, [c_void_p, c_int]),
    "ppg_run_pmbs_device": (c_int, [c_void_p, POINTER(c_double), POINTER(c_double), POINTER(PpgSearchStats),
                                    c_char_p, c_int64, POINTER(c_int64)]),
    "ppg_debug_sincos": (c_int, [c_void_p, POINTER(c_double), c_int, POINTER(c_double), POINTER(c_double)]),
    "ppg_debug_select_batch": (c_int, [c_void_p, c_int] + [c_void_p] * 7 + [c_int, c_int, c_double]
                               + [c_void_p] * 5),
    "ppg_nccl_unique_id": (c_int, [c_void_p]),
    "ppg_create_rank": (c_void_p, [c_int, c_int, c_int, c_void_p, POINTER(PpgParams), POINTER(c_int)]),
    "ppg_create_multi": (c_void_p, [c_void_p, c_int, c_int, POINTER(PpgParams), POINTER(c_int)]),
    "ppg_shard_info": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "ppg_tree_export": (c_int, [c_void_p] + [c_void_p] * 12),
    "ppg_simulate_count": (c_int, [c_void_p, POINTER(c_double), POINTER(c_int32), c_int, c_int, c_int, c_uint64,
                                   c_uint64, c_int, POINTER(c_int64), POINTER(c_int64)]),
    "ppg_measure_fp64_peak": (c_int, [c_void_p, POINTER(c_double), POINTER(c_double)]),
    "ppg_generate_cases": (c_int, [c_int, c_int, c_double, POINTER(c_uint64), c_int, POINTER(c_int32),
                                   POINTER(c_double), POINTER(c_int32), POINTER(c_double), POINTER(c_double),
                                   POINTER(c_int32), POINTER(c_int32), c_int]),
    "ppg_keyed_picks": (c_int, [c_uint64, POINTER(c_uint64), POINTER(c_uint64), POINTER(c_uint64), c_int,
                                POINTER(c_uint64)]),
}

SIMULATE_FN = ctypes.CFUNCTYPE(c_int, c_void_p, POINTER(c_double), POINTER(c_int32), c_int, c_int, c_int, c_uint64,
                               c_uint64, c_int, POINTER(c_double), POINTER(c_int64))

_LIB = None


def _torch_nccl_path():
    """The libnccl that torch ships (nvidia-nccl wheel), found without
    importing torch.  The library loads NCCL at run time; pointing it at
    torch's copy keeps one NCCL build per process whichever of the two is
    loaded first (a system libnccl.so.2 loaded before torch would shadow
    torch's by soname)."""
    try:
        import importlib.util
        spec = importlib.util.find_spec("nvidia.nccl")
    except (ImportError, ValueError):
        return None
    for d in (spec.submodule_search_locations or []) if spec else []:
        f = os.path.join(d, "lib", "libnccl.so.2")
        if os.path.exists(f):
            return f
    return None


def load_library(path: str = LIB_PATH):
    """Loads the in-tree CUDA library; raises (no fallback) when absent."""
    global _LIB
    if _LIB is not None and path == LIB_PATH:
        return _LIB
    if "PPG_NCCL_LIB" not in os.environ:
        nccl = _torch_nccl_path()
        if nccl:
            os.environ["PPG_NCCL_LIB"] = nccl
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the PMBS hot path has no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path == LIB_PATH:
        _LIB = lib
    return lib
