"""B200-native PMBS batched-rollout hot path (arxiv 2207.06649).

The device engine (libpmbs_b200.so, CUDA C++ for sm_100a) implements the
reference's batch_resolve / batch_expand / batch_simulate behind a C-ABI
(include/pushplan_gpu.h); the PMBS tree planner (run_pmbs) runs on the host in
C++ over it.  This package is the thin Python binding.
"""
from .abi import default_params, load_library  # noqa: F401
from .api import (Budget, Context, DeviceError, GraspGeometry, GraspReport, GripperTip,  # noqa: F401
                  ParallelConfig, PushResult, SearchError, SearchResult, SimError, SimParams, batch_resolve,
                  default_context, graspable, resolve_push, run_pmbs, sample_pushes)
from .world import SceneError, ShapeTable, WorldState, load_scene, scene_from_json_text, wrap_angle  # noqa: F401
