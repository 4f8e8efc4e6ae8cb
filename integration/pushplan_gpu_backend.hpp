// pushplan_gpu_backend.hpp — the REFERENCE-SIDE binding a pushplan maintainer
// adds to route the hot path through the B200 library (include/pushplan_gpu.h).
// It speaks the reference's own value types (pushplan::WorldState,
// PushAction, PushResult, pmbs::ParallelConfig) and keeps the reference's
// signatures and error behaviour, so call sites switch by replacing
//     pushplan::batch_resolve(states, pushes, tip, sim, pool)
// with
//     backend.batch_resolve(states, pushes, tip, sim)
// (and pmbs::run_pmbs(state, cfg) with backend.run_pmbs(state, cfg)).
#pragma once

#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "pushplan/pmbs.hpp"
#include "pushplan/push_sim.hpp"
#include "pushplan/world.hpp"
#include "pushplan_gpu.h"

namespace pushplan::gpu {

class BackendError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

struct PlanResult {
  PushAction action;
  mcts::SearchStats stats;
  uint64_t tree_signature_fnv = 0;  // FNV-1a of mcts::tree_signature text
  long env_steps = 0;
};

class Backend {
 public:
  explicit Backend(int device = 0);
  ~Backend();
  Backend(const Backend&) = delete;
  Backend& operator=(const Backend&) = delete;

  // push_sim.hpp:48-51 semantics: element-wise, per-element errors, SimError
  // on a length mismatch.
  std::vector<PushResult> batch_resolve(std::span<const WorldState> states, std::span<const PushAction> pushes,
                                        const GripperTip& tip, const SimParams& params);

  // pmbs.hpp:91 semantics: throws mcts::SearchError without a legal push.
  PlanResult run_pmbs(const WorldState& state, const pmbs::ParallelConfig& cfg);

 private:
  ppg_ctx* ctx_ = nullptr;
};

}  // namespace pushplan::gpu
