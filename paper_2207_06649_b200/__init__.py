"""B200-native PMBS batched-rollout hot path (arxiv 2207.06649).

The device engine (libpmbs_b200.so, CUDA C++ for sm_100a) implements the
reference's batch_resolve / batch_expand / batch_simulate behind a C-ABI
(include/pushplan_gpu.h).  run_pmbs keeps the search tree on the device by
default (csrc/dtree.cu: one CUDA-graph launch per PMBS iteration); the host
C++ tree (csrc/planner.cpp) is selectable.  Multi-GPU contexts
(Context.multi / Context.rank, csrc/multi.cu) shard the rollout batch over
GPUs with one NCCL all-reduce per wave (disc scenes) or per lockstep round.  This package is the thin
Python binding.
"""
from .abi import default_params, load_library  # noqa: F401
from .api import (Budget, Context, DeviceError, GraspGeometry, GraspReport, GripperTip, nccl_unique_id,  # noqa: F401,E501
                  ParallelConfig, PushResult, SearchError, SearchResult, SimError, SimParams, batch_resolve,
                  default_context, graspable, resolve_push, run_pmbs, sample_pushes)
from .world import SceneError, ShapeTable, WorldState, load_scene, scene_from_json_text, wrap_angle  # noqa: F401
