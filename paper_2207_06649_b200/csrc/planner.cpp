// planner.cpp — the PMBS host planner (Algorithm 1 of arxiv 2207.06649) that
// keeps the search tree on the host and drives the device through the C-ABI:
// one batched expansion (ppg_expand) and one lockstep rollout batch
// (ppg_simulate) per iteration.  Mirrors run_pmbs (pmbs.cpp:242-292) and the
// tree bookkeeping it uses (mcts.cpp:13-235, pmbs.cpp:12-131, 236-240)
// decision for decision; compiled with the reference's flags (-O3, no FMA
// contraction) so the UCB scores (glibc log/sqrt) are bit-identical.
#include <array>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "ctx.h"
#include "pushplan_gpu.h"

namespace {

using Action = std::array<double, 4>;

struct Node {
  int parent = -1;
  int depth = 0;
  double q_sum = 0.0;
  long visits = 0;
  long vvisits = 0;  // TreeNode::virtual_visits (mcts.hpp:53)
  Action action{0.0, 0.0, 0.0, 0.0};
  std::vector<Action> untried;
  size_t head = 0;  // TreeNode::untried_head (mcts.hpp:55)
  std::vector<int> children;
  bool grasp = false;
  bool dead = false;
  std::vector<double> poses;  // [n][3]
  bool terminal() const { return grasp || dead; }            // mcts.hpp:60
  bool fully_expanded() const { return head >= untried.size(); }  // mcts.hpp:61
};

struct Tree {
  std::vector<Node> nodes;  // nodes[0] is the root; children by index
  std::vector<std::vector<int>> levels;
  std::vector<int> graspable_nodes;
  int tree_depth = 7;
  int rollout_depth = 3;
  int es_level = 1;
};

constexpr double kInf = std::numeric_limits<double>::infinity();

// pmbs.cpp:12-17
double ucb_virtual(const Node& parent, const Node& child, double c) {
  const double n_child = static_cast<double>(child.visits + child.vvisits);
  if (n_child == 0.0) return kInf;
  const double n_parent = static_cast<double>(parent.visits + parent.vvisits);
  return child.q_sum / n_child + c * std::sqrt(2.0 * std::log(n_parent) / n_child);
}

// mcts.cpp:41-46
double ucb_score(const Node& parent, const Node& child, double c) {
  if (child.visits == 0) return kInf;
  const double mean = child.q_sum / static_cast<double>(child.visits);
  return mean + c * std::sqrt(2.0 * std::log(static_cast<double>(parent.visits)) /
                              static_cast<double>(child.visits));
}

// pmbs.cpp:21-28
bool subtree_selectable(const Tree& t, int id) {
  const Node& node = t.nodes[id];
  if (node.terminal()) return false;
  if (node.depth < t.tree_depth && !node.fully_expanded()) return true;
  for (int c : node.children)
    if (subtree_selectable(t, c)) return true;
  return false;
}

// pmbs.cpp:30-48
int descend_virtual(const Tree& t, double c) {
  if (!subtree_selectable(t, 0)) return -1;
  int id = 0;
  while (true) {
    const Node& node = t.nodes[id];
    if (node.depth < t.tree_depth && !node.terminal() && !node.fully_expanded()) return id;
    int best = -1;
    double best_score = -kInf;
    for (int ch : node.children) {
      if (!subtree_selectable(t, ch)) continue;
      const double score = ucb_virtual(node, t.nodes[ch], c);
      if (score > best_score) {
        best_score = score;
        best = ch;
      }
    }
    if (best < 0) return -1;
    id = best;
  }
}

// mcts.cpp:189-198
bool level_settled(const Tree& t, int level) {
  if (level < 0) return true;
  if (static_cast<size_t>(level) >= t.levels.size()) return true;
  for (int id : t.levels[level]) {
    const Node& n = t.nodes[id];
    if (n.terminal()) continue;
    if (n.depth >= t.tree_depth) continue;
    if (!n.fully_expanded()) return false;
  }
  return true;
}

// mcts.cpp:202-209
void update_es_level(Tree& t) {
  if (t.es_level > t.tree_depth) return;
  if (level_settled(t, t.es_level - 1)) ++t.es_level;
}

// mcts.cpp:211-216
bool early_stop_satisfied(const Tree& t) {
  for (int id : t.graspable_nodes)
    if (t.nodes[id].depth <= t.es_level) return true;
  return false;
}

// mcts.cpp:284-300: "depth|x_s,y_s,x_e,y_e|visits|q_sum|gd\n" pre-order,
// doubles at 17 significant digits (ostream precision(17), default format).
void signature_walk(const Tree& t, int id, std::string& out) {
  const Node& n = t.nodes[id];
  char buf[256];
  std::snprintf(buf, sizeof buf, "%d|%.17g,%.17g,%.17g,%.17g|%ld|%.17g|%c%c\n", n.depth, n.action[0],
                n.action[1], n.action[2], n.action[3], n.visits, n.q_sum, n.grasp ? 'g' : '.',
                n.dead ? 'd' : '.');
  out += buf;
  for (int c : n.children) signature_walk(t, c, out);
}

uint64_t fnv1a(const std::string& s) {
  uint64_t h = 1469598103934665603ull;
  for (unsigned char ch : s) {
    h ^= ch;
    h *= 1099511628211ull;
  }
  return h;
}

int run(ppg_ctx* ctx, const double* root_poses, double* action_out, ppg_search_stats* stats, std::string* sig) {
  const auto t_start = std::chrono::steady_clock::now();
  const auto elapsed = [&t_start] {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
  };
  const ppg_params cfg = ppg::ctx_params(ctx);
  const int n = ppg::ctx_n_objects(ctx);
  if (n <= 0) {
    ppg::ctx_set_error(ctx, "no scene installed");
    return PPG_EINVAL;
  }
  if (cfg.n_envs < 1) {
    ppg::ctx_set_error(ctx, "n_envs must be >= 1");
    return PPG_EINVAL;
  }
  const int na = cfg.pushes_per_object;
  const size_t cap_untried = static_cast<size_t>(n) * na;
  int rc;

  // SearchTree::create (mcts.cpp:28-39)
  Tree tree;
  tree.tree_depth = cfg.tree_depth;
  tree.rollout_depth = cfg.rollout_depth;
  {
    Node root;
    root.poses.assign(root_poses, root_poses + n * 3);
    std::vector<double> buf(cap_untried * 4);
    int32_t cnt = 0;
    if ((rc = ppg_sample_pushes(ctx, nullptr, root_poses, 1, buf.data(), &cnt)) != PPG_SUCCESS) return rc;
    root.untried.resize(cnt);
    std::memcpy(root.untried.data(), buf.data(), sizeof(double) * 4 * cnt);
    uint8_t g = 0;
    if ((rc = ppg_graspable(ctx, root_poses, 1, &g, nullptr, nullptr, nullptr, nullptr)) != PPG_SUCCESS) return rc;
    root.grasp = g != 0;
    root.dead = !root.grasp && root.untried.empty();
    tree.nodes.push_back(std::move(root));
    tree.levels.push_back({0});
  }
  if (tree.nodes[0].untried.empty()) {
    ppg::ctx_set_error(ctx, "no legal push action at the root");
    return PPG_ENOLEGAL;
  }

  ppg_search_stats st;
  std::memset(&st, 0, sizeof st);
  long iter = 0;
  int stop = 1;  // explored
  std::vector<int> sel_node;
  std::vector<Action> sel_action;
  std::vector<double> parent_poses, child_poses, untried, node_poses, rewards;
  std::vector<int32_t> status, n_untried, meta;
  std::vector<uint8_t> grasp;
  std::vector<int> children;
  using clk = std::chrono::steady_clock;
  const auto secs = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double>(b - a).count(); };
  while (true) {
    const auto t0 = clk::now();
    // select_batch (pmbs.cpp:52-63)
    sel_node.clear();
    sel_action.clear();
    while (static_cast<int>(sel_node.size()) < cfg.n_envs) {
      const int id = descend_virtual(tree, cfg.c_explore);
      if (id < 0) break;
      Node& node = tree.nodes[id];
      sel_action.push_back(node.untried[node.head++]);  // pop_untried mcts.cpp:13-16
      sel_node.push_back(id);
      for (int a = id; a >= 0; a = tree.nodes[a].parent) tree.nodes[a].vvisits += 1;
    }
    if (sel_node.empty()) {  // TreeExhausted
      stop = 1;
      break;
    }
    for (Node& nd : tree.nodes) nd.vvisits = 0;  // reset_virtual pmbs.cpp:65-68
    const auto t1 = clk::now();
    st.select_s += secs(t0, t1);

    // batch_expand (pmbs.cpp:70-131): device prepare, host attach in batch order
    const int P = static_cast<int>(sel_node.size());
    parent_poses.resize(static_cast<size_t>(P) * n * 3);
    for (int i = 0; i < P; ++i)
      std::memcpy(&parent_poses[static_cast<size_t>(i) * n * 3], tree.nodes[sel_node[i]].poses.data(),
                  sizeof(double) * n * 3);
    child_poses.resize(parent_poses.size());
    status.resize(P);
    grasp.resize(P);
    n_untried.resize(P);
    untried.resize(static_cast<size_t>(P) * cap_untried * 4);
    if ((rc = ppg_expand(ctx, parent_poses.data(), reinterpret_cast<const double*>(sel_action.data()), P,
                         child_poses.data(), status.data(), grasp.data(), n_untried.data(), untried.data())) !=
        PPG_SUCCESS)
      return rc;
    children.clear();
    for (int i = 0; i < P; ++i) {
      const int pid = sel_node[i];
      Node child;
      child.action = sel_action[i];
      child.parent = pid;
      child.depth = tree.nodes[pid].depth + 1;
      child.poses.assign(&child_poses[static_cast<size_t>(i) * n * 3], &child_poses[static_cast<size_t>(i + 1) * n * 3]);
      if (status[i] != PPG_OK) {
        child.dead = true;  // attach_child(nullopt) mcts.cpp:89-92
      } else {
        const double* u = &untried[static_cast<size_t>(i) * cap_untried * 4];
        child.untried.resize(n_untried[i]);
        std::memcpy(child.untried.data(), u, sizeof(double) * 4 * n_untried[i]);
        child.grasp = grasp[i] != 0;
        child.dead = !child.grasp && child.untried.empty();
      }
      const int cid = static_cast<int>(tree.nodes.size());
      const int depth = child.depth;
      const bool g = child.grasp;
      tree.nodes.push_back(std::move(child));
      tree.nodes[pid].children.push_back(cid);
      if (static_cast<size_t>(depth) >= tree.levels.size()) tree.levels.resize(depth + 1);
      tree.levels[depth].push_back(cid);
      if (g) {
        tree.graspable_nodes.push_back(cid);
        if (depth < tree.tree_depth) {
          tree.tree_depth = depth;
          tree.rollout_depth = 0;
        }
      }
      children.push_back(cid);
    }
    st.expansions += P;
    update_es_level(tree);
    const auto t2 = clk::now();
    st.expand_s += secs(t1, t2);

    // batch_simulate (pmbs.cpp:207-234) on the device
    node_poses.resize(static_cast<size_t>(P) * n * 3);
    meta.resize(static_cast<size_t>(P) * 3);
    for (int i = 0; i < P; ++i) {
      const Node& c = tree.nodes[children[i]];
      std::memcpy(&node_poses[static_cast<size_t>(i) * n * 3], c.poses.data(), sizeof(double) * n * 3);
      meta[i * 3] = c.depth;
      meta[i * 3 + 1] = c.grasp ? 1 : 0;
      meta[i * 3 + 2] = c.dead ? 1 : 0;
    }
    rewards.resize(P);
    int64_t ctr[4] = {0, 0, 0, 0};
    const ppg::SimHook hook = ppg::ctx_sim_hook(ctx);
    if (hook.fn) {
      rc = hook.fn(hook.user, node_poses.data(), meta.data(), P, cfg.n_envs, cfg.leaf_parallel, cfg.rng_seed,
                   static_cast<uint64_t>(iter), tree.tree_depth + tree.rollout_depth, rewards.data(), ctr);
    } else {
      rc = ppg_simulate(ctx, node_poses.data(), meta.data(), P, cfg.n_envs, cfg.leaf_parallel, cfg.rng_seed,
                        static_cast<uint64_t>(iter), tree.tree_depth + tree.rollout_depth, rewards.data(), ctr);
    }
    if (rc != PPG_SUCCESS) {
      if (hook.fn) ppg::ctx_set_error(ctx, "simulate hook failed");
      return rc;
    }
    const auto t3 = clk::now();
    st.simulate_s += secs(t2, t3);
    st.rollout_steps += ctr[0];
    st.lockstep_rounds += ctr[1];
    st.env_steps += ctr[3];

    // backprop_max -> backprop_mean in batch order (pmbs.cpp:236-240, mcts.cpp:180-185)
    for (int i = 0; i < P; ++i)
      for (int a = children[i]; a >= 0; a = tree.nodes[a].parent) {
        tree.nodes[a].q_sum += rewards[i];
        tree.nodes[a].visits += 1;
      }
    ++iter;
    const bool es = early_stop_satisfied(tree);
    st.backprop_s += secs(t3, clk::now());
    if (es) {
      stop = 2;
      break;
    }
    if (cfg.budget_iterations ? iter >= cfg.max_iterations : elapsed() >= cfg.max_seconds) {
      stop = 0;
      break;
    }
  }

  // best_root_child (mcts.cpp:218-235)
  const Node& root = tree.nodes[0];
  int best = -1;
  double best_score = -kInf;
  long best_visits = -1;
  for (int ch : root.children) {
    const Node& c = tree.nodes[ch];
    if (c.visits == 0) continue;
    const double score = cfg.rank_by_ucb ? ucb_score(root, c, cfg.c_explore) : c.q_sum / static_cast<double>(c.visits);
    if (score > best_score || (score == best_score && c.visits > best_visits)) {
      best_score = score;
      best_visits = c.visits;
      best = ch;
    }
  }
  if (best < 0) {
    ppg::ctx_set_error(ctx, "search produced no evaluated root child");
    return PPG_EINVAL;
  }
  std::memcpy(action_out, tree.nodes[best].action.data(), sizeof(double) * 4);
  std::string s;
  signature_walk(tree, 0, s);
  st.iterations = iter;
  st.elapsed_s = elapsed();
  st.stop_reason = stop;
  st.final_tree_depth = tree.tree_depth;
  st.env_steps += st.expansions;
  st.signature_fnv = fnv1a(s);
  st.n_nodes = static_cast<int64_t>(tree.nodes.size());
  if (stats) *stats = st;
  if (sig) *sig = std::move(s);
  return PPG_SUCCESS;
}

}  // namespace

extern "C" {

// AUTO and DEVICE: the device tree (with a simulate hook installed its
// rollouts go through the hook); HOST: this file's tree.
static bool use_device_tree(const ppg_ctx* ctx) { return ppg::ctx_planner(ctx) != PPG_PLANNER_HOST; }

int ppg_run_pmbs(ppg_ctx* ctx, const double* root_poses, double* action_out, ppg_search_stats* stats) {
  if (!ctx || !root_poses || !action_out) return PPG_EINVAL;
  if (use_device_tree(ctx)) return ppg_run_pmbs_device(ctx, root_poses, action_out, stats, nullptr, 0, nullptr);
  return run(ctx, root_poses, action_out, stats, nullptr);
}

int ppg_run_pmbs_sig(ppg_ctx* ctx, const double* root_poses, double* action_out, ppg_search_stats* stats,
                     char* sig_buf, int64_t sig_cap, int64_t* sig_len) {
  if (!ctx || !root_poses || !action_out) return PPG_EINVAL;
  if (use_device_tree(ctx)) return ppg_run_pmbs_device(ctx, root_poses, action_out, stats, sig_buf, sig_cap, sig_len);
  std::string s;
  const int rc = run(ctx, root_poses, action_out, stats, &s);
  if (rc != PPG_SUCCESS) return rc;
  if (sig_len) *sig_len = static_cast<int64_t>(s.size());
  if (sig_buf && sig_cap > 0) {
    const size_t m = s.size() < static_cast<size_t>(sig_cap - 1) ? s.size() : static_cast<size_t>(sig_cap - 1);
    std::memcpy(sig_buf, s.data(), m);
    sig_buf[m] = '\0';
  }
  return PPG_SUCCESS;
}

}  // extern "C"
