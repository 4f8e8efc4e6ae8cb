// pushplan_core_gpu.cpp — the drop-in build of the reference's pushplan::core
// whose two hot-path entry points run on the B200:
//
//   std::vector<PushResult> pushplan::batch_resolve(span<const WorldState>,
//       span<const PushAction>, const GripperTip&, const SimParams&,
//       WorkerPool*)                                       (push_sim.hpp:48-51)
//   mcts::SearchResult pushplan::pmbs::run_pmbs(const WorldState&,
//       const ParallelConfig&)                              (pmbs.hpp:91)
//
// oracle/Makefile `core_gpu` links this file with the reference's own core
// objects, in which exactly these two definitions are made weak (objcopy), so
// the unchanged callers — the reference's acceptance binary included — bind
// to the device path.  Everything else (resolve_push, sample_pushes,
// run_serial_mcts, select_batch, ...) stays the reference's.  The WorkerPool
// argument is accepted and ignored: the device replaces the pool.
#include <span>
#include <vector>

#include "pushplan/pmbs.hpp"
#include "pushplan/push_sim.hpp"
#include "pushplan_gpu_backend.hpp"

namespace pushplan {

std::vector<PushResult> batch_resolve(std::span<const WorldState> states, std::span<const PushAction> pushes,
                                      const GripperTip& tip, const SimParams& params, WorkerPool* /*pool*/) {
  return gpu::shared_backend().batch_resolve(states, pushes, tip, params);
}

namespace pmbs {

mcts::SearchResult run_pmbs(const WorldState& state, const ParallelConfig& cfg) {
  return gpu::shared_backend().run_pmbs(state, cfg);
}

}  // namespace pmbs
}  // namespace pushplan
