// adapter_check.cpp — TEST HARNESS (not product): exercises the reference-side
// binding (pushplan_gpu_backend) from inside the reference code base, the way
// the reference's acceptance criterion C8 (acceptance.cpp:372-412) checks
// batch_resolve: reference scenes and pushes, GPU batch vs the reference's own
// element-wise resolve_push, bitwise by state_digest; and run_pmbs through the
// backend vs pmbs::run_pmbs (action + tree signature FNV).
#include <cstdint>
#include <optional>
#include <string>

#include "pushplan/actions.hpp"
#include "pushplan/bench.hpp"
#include "pushplan/rng.hpp"
#include "pushplan_gpu_backend.hpp"
#include "support/scenes.hpp"

using namespace pushplan;

namespace {
uint64_t fnv(const std::string& s) {
  uint64_t h = 1469598103934665603ull;
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ull;
  }
  return h;
}
}  // namespace

extern "C" int adapter_check_c8(int target_pairs, long* pairs_out, long* mismatched_out) {
  gpu::Backend backend(0);
  const GripperTip tip;
  const SimParams sim;
  long pairs = 0, mismatched = 0;
  int k = 0;
  while (pairs < target_pairs) {
    const WorldState scene = testing::random_scene(9000 + k, 4 + k % 7);
    ++k;
    const auto pushes = sample_pushes(scene, 16, tip);
    if (pushes.empty()) continue;
    std::vector<WorldState> states(pushes.size(), scene);
    const auto batch = backend.batch_resolve(states, pushes, tip, sim);
    for (size_t i = 0; i < pushes.size(); ++i) {
      ++pairs;
      std::optional<WorldState> direct;
      try {
        direct = resolve_push(scene, pushes[i], tip, sim);
      } catch (const SimError&) {
      }
      if (direct.has_value() != batch[i].ok() ||
          (direct && state_digest(*direct) != state_digest(*batch[i].state)))
        ++mismatched;
    }
  }
  *pairs_out = pairs;
  *mismatched_out = mismatched;
  return 0;
}

extern "C" int adapter_check_pmbs(const char* case_path, const char* case_id, int* same_action, int* same_sig,
                                  int* same_stats) {
  gpu::Backend backend(0);
  const WorldState scene = load_scene(case_path);
  pmbs::ParallelConfig cfg;
  cfg.rng_seed = mix_keys(bench::episode_seed(0, case_id, 0), 0);
  const mcts::SearchResult ref = pmbs::run_pmbs(scene, cfg);
  const mcts::SearchResult got = backend.run_pmbs(scene, cfg);
  *same_action = ref.action == got.action ? 1 : 0;
  // the whole tree, rebuilt on the host from the device tree, prints the
  // reference's signature text (and its FNV equals the device's own)
  const std::string sig = mcts::tree_signature(*got.tree);
  *same_sig = (sig == mcts::tree_signature(*ref.tree) && fnv(sig) == backend.last_device_stats().signature_fnv) ? 1 : 0;
  *same_stats = (ref.stats.iterations == got.stats.iterations && ref.stats.expansions == got.stats.expansions &&
                 ref.stats.stop_reason == got.stats.stop_reason)
                    ? 1
                    : 0;
  return 0;
}
