// pushplan_gpu_backend.cpp — see the header.  Marshals reference value types
// into the flat C-ABI arrays and back.
#include "pushplan_gpu_backend.hpp"

#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <tuple>

namespace pushplan::gpu {

namespace {

ppg_params to_params(const GripperTip& tip, const SimParams& sim) {
  ppg_params p;
  ppg_params_default(&p);
  p.tip_radius = tip.radius;
  p.tip_clearance = tip.clearance;
  p.push_distance = sim.push_distance;
  p.substeps = sim.substeps;
  p.max_projection_iters = sim.max_projection_iters;
  p.eps_pen = sim.eps_pen;
  p.rotation_gain = sim.rotation_gain;
  return p;
}

struct Flat {
  std::vector<int32_t> kind, nv, target;
  std::vector<double> radius, verts, poses;
  bool any_polygon = false;
  void add(const WorldState& s) {
    target.push_back(s.target_index);
    for (const PlacedObject& o : s.objects) {
      const bool disc = o.shape.kind == ObjectShape::Kind::Disc;
      any_polygon = any_polygon || !disc;
      kind.push_back(disc ? PPG_DISC : PPG_POLYGON);
      radius.push_back(o.shape.radius);
      nv.push_back(static_cast<int32_t>(o.shape.vertices.size()));
      for (int k = 0; k < PPG_MAX_VERTICES; ++k) {
        const bool ok = k < static_cast<int>(o.shape.vertices.size());
        verts.push_back(ok ? o.shape.vertices[k].x : 0.0);
        verts.push_back(ok ? o.shape.vertices[k].y : 0.0);
      }
      poses.push_back(o.pose.x);
      poses.push_back(o.pose.y);
      poses.push_back(o.pose.theta);
    }
  }
  ppg_shapes shapes(int n, int tables, const Workspace& ws) const {
    ppg_shapes sh;
    sh.n_objects = n;
    sh.n_tables = tables;
    sh.kind = kind.data();
    sh.radius = radius.data();
    sh.n_vertices = any_polygon ? nv.data() : nullptr;
    sh.vertices = any_polygon ? verts.data() : nullptr;
    sh.target_index = target.data();
    sh.side_length = ws.side_length;
    sh.boundary_margin = ws.boundary_margin;
    return sh;
  }
};

}  // namespace

Backend::Backend(int device) {
  int err = 0;
  ctx_ = ppg_create(device, nullptr, &err);
  if (!ctx_) throw BackendError("ppg_create failed (code " + std::to_string(err) + ")");
}

Backend::~Backend() { ppg_destroy(ctx_); }

std::vector<PushResult> Backend::batch_resolve(std::span<const WorldState> states,
                                               std::span<const PushAction> pushes, const GripperTip& tip,
                                               const SimParams& params) {
  if (states.size() != pushes.size()) throw SimError("batch_resolve: states and pushes must have equal length");
  std::vector<PushResult> results(states.size());
  ppg_params p = to_params(tip, params);
  if (ppg_set_params(ctx_, &p) != PPG_SUCCESS) throw BackendError(ppg_last_error(ctx_));
  // one launch per (object count, workspace): the C-ABI takes uniform batches
  std::map<std::tuple<size_t, double, double>, std::vector<size_t>> groups;
  for (size_t i = 0; i < states.size(); ++i)
    groups[{states[i].objects.size(), states[i].workspace.side_length, states[i].workspace.boundary_margin}]
        .push_back(i);
  for (const auto& [key, idx] : groups) {
    const int n = static_cast<int>(std::get<0>(key));
    Flat f;
    std::vector<double> acts;
    for (size_t i : idx) {
      f.add(states[i]);
      const PushAction& a = pushes[i];
      acts.insert(acts.end(), {a.x_s, a.y_s, a.x_e, a.y_e});
    }
    const int E = static_cast<int>(idx.size());
    const ppg_shapes sh = f.shapes(n, E, states[idx[0]].workspace);
    std::vector<double> out(f.poses.size());
    std::vector<int32_t> status(E);
    std::vector<double> resid(E);
    if (ppg_batch_resolve(ctx_, &sh, f.poses.data(), acts.data(), E, out.data(), status.data(), resid.data()) !=
        PPG_SUCCESS)
      throw BackendError(ppg_last_error(ctx_));
    for (int k = 0; k < E; ++k) {
      PushResult& r = results[idx[k]];
      if (status[k] == PPG_OK) {
        WorldState s = states[idx[k]];
        for (int o = 0; o < n; ++o) {
          s.objects[o].pose.x = out[(static_cast<size_t>(k) * n + o) * 3];
          s.objects[o].pose.y = out[(static_cast<size_t>(k) * n + o) * 3 + 1];
          s.objects[o].pose.theta = out[(static_cast<size_t>(k) * n + o) * 3 + 2];
        }
        r.state = std::move(s);
      } else if (status[k] == PPG_START_COLLISION) {
        r.error = "resolve_push: gripper start pose collides or leaves the workspace";
      } else {
        std::ostringstream msg;  // the reference's own formatting (push_sim.cpp:124-126)
        msg << "resolve_push: projection did not converge, residual penetration " << resid[k] << " m";
        r.error = msg.str();
      }
    }
  }
  return results;
}

mcts::SearchResult Backend::run_pmbs(const WorldState& state, const pmbs::ParallelConfig& cfg) {
  ppg_params p = to_params(cfg.tip, cfg.sim);
  p.finger_width = cfg.grasp.finger_width;
  p.finger_thickness = cfg.grasp.finger_thickness;
  p.opening = cfg.grasp.opening;
  p.approach_clearance = cfg.grasp.approach_clearance;
  p.gamma = cfg.gamma;
  p.c_explore = cfg.c_explore;
  p.tree_depth = cfg.tree_depth;
  p.rollout_depth = cfg.rollout_depth;
  p.pushes_per_object = cfg.pushes_per_object;
  p.margin_threshold = cfg.margin_threshold;
  p.rng_seed = cfg.rng_seed;
  p.rank_by_ucb = cfg.rank_by_ucb ? 1 : 0;
  p.budget_iterations = cfg.budget.mode == mcts::Budget::Mode::Iterations ? 1 : 0;
  p.max_iterations = cfg.budget.max_iterations;
  p.max_seconds = cfg.budget.max_seconds;
  p.n_envs = cfg.n_envs;
  p.leaf_parallel = cfg.leaf_parallel ? 1 : 0;
  if (ppg_set_params(ctx_, &p) != PPG_SUCCESS) throw BackendError(ppg_last_error(ctx_));
  Flat f;
  f.add(state);
  const int n = static_cast<int>(state.objects.size());
  const ppg_shapes sh = f.shapes(n, 1, state.workspace);
  if (ppg_set_scene(ctx_, &sh) != PPG_SUCCESS) throw BackendError(ppg_last_error(ctx_));
  double action[4];
  const int rc = ppg_run_pmbs(ctx_, f.poses.data(), action, &last_);
  // the reference's messages (mcts.cpp:244, pmbs.cpp:248)
  if (rc == PPG_ENOLEGAL) throw mcts::SearchError("no legal push action at the root");
  if (rc != PPG_SUCCESS) throw BackendError(ppg_last_error(ctx_));
  mcts::SearchResult r;
  r.action = PushAction{action[0], action[1], action[2], action[3]};
  r.stats.iterations = last_.iterations;
  r.stats.expansions = last_.expansions;
  r.stats.elapsed_s = last_.elapsed_s;
  r.stats.stop_reason = last_.stop_reason == 0 ? "budget" : (last_.stop_reason == 1 ? "explored" : "early_stop");
  // the tree: one export of the device tree's node arrays
  int64_t N = 0, U = 0;
  if (ppg_tree_export(ctx_, &N, &U, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                      nullptr) != PPG_SUCCESS)
    throw BackendError(ppg_last_error(ctx_));
  std::vector<int32_t> parent(N), depth(N), ucount(N), scal(4);
  std::vector<double> act(N * 4), q(N), poses(N * n * 3), untried(U * 4);
  std::vector<int64_t> visits(N);
  std::vector<uint8_t> flags(N);
  if (ppg_tree_export(ctx_, &N, &U, parent.data(), depth.data(), act.data(), visits.data(), q.data(), flags.data(),
                      poses.data(), ucount.data(), untried.data(), scal.data()) != PPG_SUCCESS)
    throw BackendError(ppg_last_error(ctx_));
  auto tree = std::make_unique<mcts::SearchTree>();
  std::vector<mcts::TreeNode*> node(N, nullptr);
  size_t uk = 0;
  for (int64_t x = 0; x < N; ++x) {
    std::unique_ptr<mcts::TreeNode> own = std::make_unique<mcts::TreeNode>();
    mcts::TreeNode* t = own.get();
    t->state = state;
    for (int o = 0; o < n; ++o) {
      t->state.objects[o].pose.x = poses[(x * n + o) * 3];
      t->state.objects[o].pose.y = poses[(x * n + o) * 3 + 1];
      t->state.objects[o].pose.theta = poses[(x * n + o) * 3 + 2];
    }
    t->action = PushAction{act[x * 4], act[x * 4 + 1], act[x * 4 + 2], act[x * 4 + 3]};
    t->depth = depth[x];
    t->q_sum = q[x];
    t->visits = static_cast<long>(visits[x]);
    t->graspable_flag = (flags[x] & 1) != 0;
    t->dead_flag = (flags[x] & 2) != 0;
    for (int k = 0; k < ucount[x]; ++k, ++uk)
      t->untried.push_back(PushAction{untried[uk * 4], untried[uk * 4 + 1], untried[uk * 4 + 2], untried[uk * 4 + 3]});
    if (static_cast<size_t>(t->depth) >= tree->levels.size()) tree->levels.resize(t->depth + 1);
    tree->levels[t->depth].push_back(t);
    if (t->graspable_flag) tree->graspable_nodes.push_back(t);
    node[x] = t;
    if (x == 0) {
      tree->root = std::move(own);
    } else {
      t->parent = node[parent[x]];
      t->parent->children.push_back(std::move(own));
    }
  }
  tree->tree_depth = scal[0];
  tree->rollout_depth = scal[1];
  tree->es_level = scal[2];
  r.tree = std::move(tree);
  return r;
}

Backend& shared_backend() {
  static std::unique_ptr<Backend> b;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* d = std::getenv("PPG_DEVICE");
    b = std::make_unique<Backend>(d ? std::atoi(d) : 0);
  });
  return *b;
}

}  // namespace pushplan::gpu
