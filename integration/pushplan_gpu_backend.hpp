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
  // The returned SearchResult carries the whole search tree (rebuilt on the
  // host from the device-resident tree, ppg_tree_export), so callers of
  // mcts::tree_signature(*result.tree) work unchanged.
  mcts::SearchResult run_pmbs(const WorldState& state, const pmbs::ParallelConfig& cfg);

  // Device-side statistics of the last run_pmbs (not in mcts::SearchStats).
  const ppg_search_stats& last_device_stats() const { return last_; }

 private:
  ppg_ctx* ctx_ = nullptr;
  ppg_search_stats last_{};
};

// The process-wide backend used by pushplan_core_gpu (the drop-in build of
// pushplan::core whose batch_resolve / pmbs::run_pmbs run on the device);
// device from PPG_DEVICE (default 0).
Backend& shared_backend();

}  // namespace pushplan::gpu
