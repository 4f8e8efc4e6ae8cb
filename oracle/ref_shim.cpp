// ref_shim.cpp — TEST INFRASTRUCTURE ONLY (oracle).  Never linked into the
// product.  A flat C-ABI over the UNMODIFIED reference library compiled from
// /root/reference/proj/core/src by oracle/Makefile into oracle/_ref/.  It lets
// the pytest parity suite, the golden-fixture generator and bench.py's
// reference / cpu_baseline arm call the reference's own public API
// (batch_resolve, sample_pushes, graspable, run_pmbs, generate_case, ...)
// on the same flat arrays the product C-ABI (include/pushplan_gpu.h) takes.
#include <chrono>
#include <cmath>
#include <cstring>
#include <fstream>
#include <functional>
#include <sstream>
#include <memory>
#include <random>
#include <string>
#include <vector>

#include "pushplan/actions.hpp"
#include "pushplan/bench.hpp"
#include "pushplan/mcts.hpp"
#include "pushplan/pmbs.hpp"
#include "pushplan/push_sim.hpp"
#include "pushplan/rng.hpp"
#include "pushplan/worker_pool.hpp"
#include "pushplan/world.hpp"
#include "pushplan_gpu.h"
#include "support/scenes.hpp"

using namespace pushplan;

namespace {

struct States {
  std::vector<WorldState> v;
  std::vector<PushResult> results;
};

pmbs::ParallelConfig to_cfg(const ppg_params* p) {
  pmbs::ParallelConfig c;
  c.tip.radius = p->tip_radius;
  c.tip.clearance = p->tip_clearance;
  c.sim.push_distance = p->push_distance;
  c.sim.substeps = p->substeps;
  c.sim.max_projection_iters = p->max_projection_iters;
  c.sim.eps_pen = p->eps_pen;
  c.sim.rotation_gain = p->rotation_gain;
  c.grasp.finger_width = p->finger_width;
  c.grasp.finger_thickness = p->finger_thickness;
  c.grasp.opening = p->opening;
  c.grasp.approach_clearance = p->approach_clearance;
  c.gamma = p->gamma;
  c.c_explore = p->c_explore;
  c.tree_depth = p->tree_depth;
  c.rollout_depth = p->rollout_depth;
  c.pushes_per_object = p->pushes_per_object;
  c.margin_threshold = p->margin_threshold;
  c.rng_seed = p->rng_seed;
  c.rank_by_ucb = p->rank_by_ucb != 0;
  c.budget = p->budget_iterations ? mcts::Budget::iterations(p->max_iterations)
                                  : mcts::Budget::seconds(p->max_seconds);
  c.n_envs = p->n_envs;
  c.leaf_parallel = p->leaf_parallel != 0;
  return c;
}

uint64_t fnv(const std::string& s) {
  uint64_t h = 1469598103934665603ull;
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ull;
  }
  return h;
}

int stop_code(const std::string& s) {
  if (s == "budget") return 0;
  if (s == "explored") return 1;
  return 2;
}

}  // namespace

extern "C" {

void* ref_states_new(const ppg_shapes* sh, const double* poses, int E) {
  auto* st = new States;
  st->v.resize(E);
  const int n = sh->n_objects;
  for (int e = 0; e < E; ++e) {
    const int t = sh->n_tables == 1 ? 0 : e;
    WorldState& w = st->v[e];
    w.workspace.side_length = sh->side_length;
    w.workspace.boundary_margin = sh->boundary_margin;
    w.target_index = sh->target_index[t];
    w.objects.resize(n);
    for (int i = 0; i < n; ++i) {
      PlacedObject& o = w.objects[i];
      const int s = t * n + i;
      if (sh->kind[s] == PPG_DISC) {
        o.shape = ObjectShape::disc(sh->radius[s]);
      } else {
        Polygon verts;
        for (int k = 0; k < sh->n_vertices[s]; ++k)
          verts.push_back({sh->vertices[(s * PPG_MAX_VERTICES + k) * 2],
                           sh->vertices[(s * PPG_MAX_VERTICES + k) * 2 + 1]});
        o.shape = ObjectShape::polygon(verts);
      }
      o.pose.x = poses[(e * n + i) * 3];
      o.pose.y = poses[(e * n + i) * 3 + 1];
      o.pose.theta = poses[(e * n + i) * 3 + 2];
    }
  }
  return st;
}

void ref_states_free(void* h) { delete static_cast<States*>(h); }
int ref_states_count(void* h) { return static_cast<int>(static_cast<States*>(h)->v.size()); }
int ref_state_n(void* h, int i) {
  return static_cast<int>(static_cast<States*>(h)->v.at(i).objects.size());
}

// Exports state i: arrays sized n, n, n, n*MAXV*2, n*3.
int ref_state_export(void* h, int i, int32_t* kind, double* radius, int32_t* nverts,
                     double* verts, double* poses, int32_t* target, double* side,
                     double* margin) {
  const WorldState& w = static_cast<States*>(h)->v.at(i);
  const int n = static_cast<int>(w.objects.size());
  for (int k = 0; k < n; ++k) {
    const PlacedObject& o = w.objects[k];
    kind[k] = o.shape.kind == ObjectShape::Kind::Disc ? PPG_DISC : PPG_POLYGON;
    radius[k] = o.shape.radius;
    nverts[k] = static_cast<int32_t>(o.shape.vertices.size());
    for (int v = 0; v < PPG_MAX_VERTICES; ++v) {
      const bool ok = v < static_cast<int>(o.shape.vertices.size());
      verts[(k * PPG_MAX_VERTICES + v) * 2] = ok ? o.shape.vertices[v].x : 0.0;
      verts[(k * PPG_MAX_VERTICES + v) * 2 + 1] = ok ? o.shape.vertices[v].y : 0.0;
    }
    poses[k * 3] = o.pose.x;
    poses[k * 3 + 1] = o.pose.y;
    poses[k * 3 + 2] = o.pose.theta;
  }
  *target = w.target_index;
  *side = w.workspace.side_length;
  *margin = w.workspace.boundary_margin;
  return n;
}

// bench::generate_case (bench.cpp:234-259); motif 0 random, 1 ring, 2 wall
// (bench.cpp:261-317).  Returns NULL on BenchError.
void* ref_generate_case(int motif, int n_objects, double polygon_fraction, uint64_t seed) {
  try {
    auto* st = new States;
    st->v.push_back(bench::generate_case_motif(static_cast<bench::Motif>(motif), n_objects,
                                               bench::ShapeMix{polygon_fraction}, seed));
    return st;
  } catch (const std::exception&) {
    return nullptr;
  }
}

// BASELINE config 2 inputs built by the reference alone (bench.py's
// reference arm and the full-workload parity test): scene k =
// bench::generate_case(n, ShapeMix{pf}, seed) for consecutive seeds from
// seed_base, skipping seeds whose generator throws and scenes with no legal
// push (sample_pushes(scene, N_a)); push k = that list's
// uniform_int_distribution pick from keyed_rng(pick_seed, k, 0)
// (rng.hpp:21-23, mcts.cpp:151-152).  Same rule as the product's
// scenes.c2_workload.  Scenes are generated by `threads` threads.
void* ref_c2_workload(int n_objects, double polygon_fraction, uint64_t seed_base, int E, uint64_t pick_seed,
                      int pushes_per_object, int threads, double* pushes_out, uint64_t* seeds_out) {
  GripperTip tip;
  const int batch = E + E / 16 + 64;
  auto* st = new States;
  uint64_t next = seed_base;
  int k = 0;
  while (k < E) {
    std::vector<std::unique_ptr<WorldState>> gen(batch);
    std::vector<std::vector<PushAction>> cand(batch);
    const uint64_t base = next;
    WorkerPool pool(threads > 1 ? threads : 1);
    pool.parallel_for(batch, [&](int i) {
      try {
        gen[i] = std::make_unique<WorldState>(bench::generate_case(n_objects, bench::ShapeMix{polygon_fraction},
                                                                   base + static_cast<uint64_t>(i)));
        cand[i] = sample_pushes(*gen[i], pushes_per_object, tip);
      } catch (const std::exception&) {
        gen[i].reset();
      }
    });
    next += static_cast<uint64_t>(batch);
    for (int i = 0; i < batch && k < E; ++i) {
      if (!gen[i] || cand[i].empty()) continue;
      auto rng = keyed_rng(pick_seed, static_cast<uint64_t>(k), 0);
      std::uniform_int_distribution<size_t> pick(0, cand[i].size() - 1);
      const PushAction& a = cand[i][pick(rng)];
      pushes_out[k * 4] = a.x_s;
      pushes_out[k * 4 + 1] = a.y_s;
      pushes_out[k * 4 + 2] = a.x_e;
      pushes_out[k * 4 + 3] = a.y_e;
      if (seeds_out) seeds_out[k] = base + static_cast<uint64_t>(i);
      st->v.push_back(std::move(*gen[i]));
      ++k;
    }
  }
  return st;
}

// Acceptance criterion 3 (acceptance.cpp:255-281): 200 select_batch
// invocations on random explicit trees.  random_tree (acceptance.cpp:64-92)
// is restated here with the same libstdc++ distributions and draw order (the
// reference keeps it file-local to its acceptance binary); select_batch and
// reset_virtual are the reference's own (pmbs.cpp:52-68).  variant 0 is the
// criterion exactly (rng keyed_rng(3, 0, 0) shared by the 200 trees,
// n_envs = {4, 16, 64}[t % 3], tree_depth 7); variant 1 additionally marks
// nodes terminal (graspable / dead) from keyed_rng(4, t, 0) and uses
// tree_depth 1 + t % 4, so the selectable-subtree logic and TreeExhausted are
// exercised too.  Per tree t, nodes in pre-order (children in insertion
// order) go to the flat arrays from node_off[t]; the selected pairs (node
// index, popped untried index) from pair_off[t]; vv = virtual visits after
// select_batch, before reset_virtual; vsum = sum of virtual visits after it.
int ref_c3_trees(int variant, int count, int cap_nodes, int cap_pairs, int32_t* node_off, int32_t* parent,
                 int32_t* depth, int64_t* visits, double* q_sum, uint8_t* flags, int32_t* n_children,
                 int32_t* n_untried, int64_t* vv, int32_t* pair_off, int32_t* sel_node, int32_t* sel_untried,
                 int32_t* tree_depth, int32_t* n_envs, int64_t* vsum, int32_t* exhausted) {
  auto rng = keyed_rng(3, 0, 0);
  int tag = 0;
  const auto synth = [&tag] {
    const int i = ++tag;
    return PushAction{1e-4 * i, 2e-4 * i, 1e-4 * i + 0.05, 2e-4 * i};
  };
  int nn = 0, np = 0;
  const int env_choices[3] = {4, 16, 64};
  for (int t = 0; t < count; ++t) {
    std::uniform_int_distribution<int> kids(0, 3);
    std::uniform_int_distribution<long> vis(1, 20);
    std::uniform_real_distribution<double> uq(0.0, 1.0);
    std::uniform_int_distribution<int> untried(0, 2);
    const std::function<void(mcts::TreeNode&, int)> grow = [&](mcts::TreeNode& node, int d) {
      const int n = d < 4 ? kids(rng) : 0;
      long total = vis(rng);
      for (int i = 0; i < n; ++i) {
        auto child = std::make_unique<mcts::TreeNode>();
        child->action = synth();
        child->parent = &node;
        child->depth = node.depth + 1;
        grow(*child, d + 1);
        total += child->visits;
        node.children.push_back(std::move(child));
      }
      node.visits = total;
      node.q_sum = uq(rng) * static_cast<double>(total);
      const int u = untried(rng);
      for (int i = 0; i < u; ++i) node.untried.push_back(synth());
    };
    mcts::SearchTree tree;
    tree.root = std::make_unique<mcts::TreeNode>();
    grow(*tree.root, 0);
    if (tree.root->untried.empty()) tree.root->untried.push_back(synth());
    pmbs::ParallelConfig cfg;
    cfg.n_envs = env_choices[t % 3];
    if (variant == 1) {
      tree.tree_depth = 1 + t % 4;
      auto r2 = keyed_rng(4, static_cast<uint64_t>(t), 0);
      std::uniform_int_distribution<int> pick(0, 19);
      const std::function<void(mcts::TreeNode&)> mark = [&](mcts::TreeNode& x) {
        const int v = pick(r2);
        if (x.parent && v == 0) x.graspable_flag = true;
        else if (x.parent && v == 1) x.dead_flag = true;
        for (auto& c : x.children) mark(*c);
      };
      mark(*tree.root);
    }
    // pre-order numbering
    std::vector<mcts::TreeNode*> order;
    const std::function<void(mcts::TreeNode&)> walk = [&](mcts::TreeNode& x) {
      order.push_back(&x);
      for (auto& c : x.children) walk(*c);
    };
    walk(*tree.root);
    if (nn + static_cast<int>(order.size()) > cap_nodes) return -1;
    node_off[t] = nn;
    std::vector<std::pair<mcts::TreeNode*, int>> idx;
    for (size_t k = 0; k < order.size(); ++k) {
      mcts::TreeNode* x = order[k];
      int pi = -1;
      for (size_t m = 0; m < k; ++m)
        if (order[m] == x->parent) pi = static_cast<int>(m);
      parent[nn + k] = pi;
      depth[nn + k] = x->depth;
      visits[nn + k] = x->visits;
      q_sum[nn + k] = x->q_sum;
      flags[nn + k] = static_cast<uint8_t>((x->graspable_flag ? 1 : 0) | (x->dead_flag ? 2 : 0));
      n_children[nn + k] = static_cast<int32_t>(x->children.size());
      n_untried[nn + k] = static_cast<int32_t>(x->untried.size());
    }
    tree_depth[t] = tree.tree_depth;
    n_envs[t] = cfg.n_envs;
    pair_off[t] = np;
    exhausted[t] = 0;
    try {
      const pmbs::SelectionBatch batch = pmbs::select_batch(tree, cfg);
      if (np + static_cast<int>(batch.pairs.size()) > cap_pairs) return -2;
      std::vector<size_t> popped(order.size(), 0);
      for (const auto& [node, action] : batch.pairs) {
        size_t k = 0;
        while (order[k] != node) ++k;
        sel_node[np] = static_cast<int32_t>(k);
        sel_untried[np] = static_cast<int32_t>(popped[k]++);
        ++np;
      }
    } catch (const pmbs::TreeExhausted&) {
      exhausted[t] = 1;
    }
    for (size_t k = 0; k < order.size(); ++k) vv[nn + k] = order[k]->virtual_visits;
    pmbs::reset_virtual(*tree.root);
    long sum = 0;
    for (mcts::TreeNode* x : order) sum += x->virtual_visits;
    vsum[t] = sum;
    nn += static_cast<int>(order.size());
  }
  node_off[count] = nn;
  pair_off[count] = np;
  return 0;
}

void* ref_load_scene(const char* path) {
  try {
    auto* st = new States;
    st->v.push_back(load_scene(path));
    return st;
  } catch (const std::exception&) {
    return nullptr;
  }
}

// Test-support fixtures (tests/support/scenes.cpp:34-95).
void* ref_fixture(const char* name, double arg, int iarg) {
  auto* st = new States;
  const std::string s(name);
  try {
    if (s == "lone_disc") st->v.push_back(testing::lone_disc(arg));
    else if (s == "two_discs_row") st->v.push_back(testing::two_discs_row(arg));
    else if (s == "hex_ring") st->v.push_back(testing::hex_ring());
    else if (s == "arc_ring") st->v.push_back(testing::arc_ring());
    else if (s == "arc_ring_open") st->v.push_back(testing::arc_ring_open());
    else if (s == "corridor") st->v.push_back(testing::corridor_scene());
    else if (s == "packed_clutter") st->v.push_back(testing::packed_clutter());
    else if (s == "random_scene") st->v.push_back(testing::random_scene(static_cast<uint64_t>(arg), iarg));
    else if (s == "search_case") st->v.push_back(testing::search_case(static_cast<uint64_t>(arg), iarg));
    else {
      delete st;
      return nullptr;
    }
  } catch (const std::exception&) {
    delete st;
    return nullptr;
  }
  return st;
}

// acceptance.cpp:124-134 deep_search_case: a random scene that is not
// graspable, has legal pushes and no winning first push.
void* ref_deep_search_case(uint64_t seed, int n_objects) {
  mcts::SearchConfig probe;
  for (uint64_t k = 0; k < 2000; ++k) {
    const WorldState s = testing::random_scene(mix_keys(seed, k), n_objects);
    if (graspable(s, probe.grasp, probe.margin_threshold).graspable) continue;
    if (sample_pushes(s, probe.pushes_per_object, probe.tip).empty()) continue;
    if (!testing::winning_first_pushes(s, probe, 1).empty()) continue;
    auto* st = new States;
    st->v.push_back(s);
    return st;
  }
  return nullptr;
}

uint64_t ref_state_digest(void* h, int i) {
  return state_digest(static_cast<States*>(h)->v.at(i));
}

// Times pushplan::batch_resolve alone (push_sim.cpp:132-152) with a
// WorkerPool of `threads` (<= 1: pool == nullptr, inline).  Results stay in
// the handle; ref_batch_results copies them out.
int ref_batch_resolve(void* h, const double* pushes, const ppg_params* p, int threads,
                      double* seconds) {
  States* st = static_cast<States*>(h);
  const size_t E = st->v.size();
  std::vector<PushAction> acts(E);
  for (size_t e = 0; e < E; ++e)
    acts[e] = {pushes[e * 4], pushes[e * 4 + 1], pushes[e * 4 + 2], pushes[e * 4 + 3]};
  GripperTip tip{p->tip_radius, p->tip_clearance};
  SimParams sim;
  sim.push_distance = p->push_distance;
  sim.substeps = p->substeps;
  sim.max_projection_iters = p->max_projection_iters;
  sim.eps_pen = p->eps_pen;
  sim.rotation_gain = p->rotation_gain;
  std::unique_ptr<WorkerPool> pool;
  if (threads > 1) pool = std::make_unique<WorkerPool>(threads);
  const auto t0 = std::chrono::steady_clock::now();
  st->results = batch_resolve(st->v, acts, tip, sim, pool.get());
  const auto t1 = std::chrono::steady_clock::now();
  if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
  return 0;
}

// status: 0 ok, 1 start collision, 2 non-converged (message text classifies).
int ref_batch_results(void* h, double* poses_out, int32_t* status, uint64_t* digests) {
  States* st = static_cast<States*>(h);
  for (size_t e = 0; e < st->results.size(); ++e) {
    const PushResult& r = st->results[e];
    const int n = static_cast<int>(st->v[e].objects.size());
    if (r.ok()) {
      status[e] = PPG_OK;
      for (int i = 0; i < n; ++i) {
        poses_out[(e * n + i) * 3] = r.state->objects[i].pose.x;
        poses_out[(e * n + i) * 3 + 1] = r.state->objects[i].pose.y;
        poses_out[(e * n + i) * 3 + 2] = r.state->objects[i].pose.theta;
      }
      if (digests) digests[e] = state_digest(*r.state);
    } else {
      status[e] = r.error.find("collides") != std::string::npos ? PPG_START_COLLISION
                                                                : PPG_NOT_CONVERGED;
      for (int i = 0; i < n * 3; ++i) poses_out[e * n * 3 + i] = 0.0;
      if (digests) digests[e] = 0;
    }
  }
  return 0;
}

int ref_sample_pushes(void* h, int i, const ppg_params* p, double* out, int cap) {
  const WorldState& w = static_cast<States*>(h)->v.at(i);
  const auto v = sample_pushes(w, p->pushes_per_object, GripperTip{p->tip_radius, p->tip_clearance},
                               p->push_distance);
  const int n = static_cast<int>(v.size());
  for (int k = 0; k < n && k < cap; ++k) {
    out[k * 4] = v[k].x_s;
    out[k * 4 + 1] = v[k].y_s;
    out[k * 4 + 2] = v[k].x_e;
    out[k * 4 + 3] = v[k].y_e;
  }
  return n;
}

int ref_graspable(void* h, int i, const ppg_params* p, double* margin, double* best_x,
                  double* best_y, int32_t* best_angle) {
  const WorldState& w = static_cast<States*>(h)->v.at(i);
  GraspGeometry g;
  g.finger_width = p->finger_width;
  g.finger_thickness = p->finger_thickness;
  g.opening = p->opening;
  g.approach_clearance = p->approach_clearance;
  const GraspReport r = graspable(w, g, p->margin_threshold);
  *margin = r.margin;
  if (r.best) {
    *best_x = r.best->x;
    *best_y = r.best->y;
    *best_angle = r.best->angle_index;
  } else {
    *best_x = 0.0;
    *best_y = 0.0;
    *best_angle = -1;
  }
  return r.graspable ? 1 : 0;
}

// `count` uniform picks in [0, n) from keyed_rng(seed, iter, env) through
// std::uniform_int_distribution<size_t> (mcts.cpp:151-152).
int ref_keyed_picks(uint64_t seed, uint64_t iter, uint64_t env, int count, uint64_t n,
                    uint64_t* out) {
  std::mt19937_64 rng = keyed_rng(seed, iter, env);
  for (int k = 0; k < count; ++k) {
    std::uniform_int_distribution<size_t> pick(0, n - 1);
    out[k] = pick(rng);
  }
  return 0;
}

int ref_keyed_raw(uint64_t seed, uint64_t iter, uint64_t env, int count, uint64_t* out) {
  std::mt19937_64 rng = keyed_rng(seed, iter, env);
  for (int k = 0; k < count; ++k) out[k] = rng();
  return 0;
}

uint64_t ref_mix_keys(uint64_t seed, uint64_t a, uint64_t b) { return mix_keys(seed, a, b); }

uint64_t ref_episode_seed(uint64_t base, const char* case_id, int trial) {
  return bench::episode_seed(base, case_id, trial);
}

// run_pmbs (pmbs.cpp:242-292) or run_serial_mcts (mcts.cpp:237-282).
int ref_run_search(void* h, int i, const ppg_params* p, int threads, int serial,
                   double* action, ppg_search_stats* stats, char* sig_buf, int64_t sig_cap,
                   int64_t* sig_len) {
  const WorldState& w = static_cast<States*>(h)->v.at(i);
  pmbs::ParallelConfig cfg = to_cfg(p);
  cfg.worker_threads = threads;
  mcts::SearchResult r;
  try {
    r = serial ? mcts::run_serial_mcts(w, cfg) : pmbs::run_pmbs(w, cfg);
  } catch (const mcts::SearchError&) {
    return PPG_ENOLEGAL;
  }
  action[0] = r.action.x_s;
  action[1] = r.action.y_s;
  action[2] = r.action.x_e;
  action[3] = r.action.y_e;
  const std::string sig = mcts::tree_signature(*r.tree);
  std::memset(stats, 0, sizeof *stats);
  stats->iterations = r.stats.iterations;
  stats->expansions = r.stats.expansions;
  stats->elapsed_s = r.stats.elapsed_s;
  stats->stop_reason = stop_code(r.stats.stop_reason);
  stats->final_tree_depth = r.tree->tree_depth;
  stats->signature_fnv = fnv(sig);
  long nodes = 0;
  for (const auto& lvl : r.tree->levels) nodes += static_cast<long>(lvl.size());
  stats->n_nodes = nodes;
  if (sig_len) *sig_len = static_cast<int64_t>(sig.size());
  if (sig_buf && sig_cap > 0) {
    const size_t m = std::min<size_t>(sig.size(), static_cast<size_t>(sig_cap - 1));
    std::memcpy(sig_buf, sig.data(), m);
    sig_buf[m] = '\0';
  }
  return 0;
}

// First PMBS iteration of a search on state i, exposed piecewise so the
// device lockstep engine can be checked against the reference's own
// batch_simulate on identical children: SearchTree::create -> select_batch ->
// reset_virtual -> batch_expand -> update_es_level -> batch_simulate(iteration).
// Outputs: n_children; child poses [N][n][3]; meta [N][3] = depth, graspable,
// dead; rewards [N]; depth_cap.
int ref_first_iteration(void* h, int i, const ppg_params* p, uint64_t iteration,
                        double* child_poses, int32_t* meta, double* rewards,
                        int32_t* depth_cap) {
  const WorldState& w = static_cast<States*>(h)->v.at(i);
  pmbs::ParallelConfig cfg = to_cfg(p);
  mcts::SearchTree tree = mcts::SearchTree::create(w, cfg);
  if (tree.root->untried.empty()) return -1;
  pmbs::SelectionBatch batch = pmbs::select_batch(tree, cfg);
  pmbs::reset_virtual(*tree.root);
  const auto children = pmbs::batch_expand(tree, batch, cfg, nullptr);
  mcts::update_es_level(tree);
  const auto r = pmbs::batch_simulate(tree, children, cfg, nullptr, iteration);
  const int n = static_cast<int>(w.objects.size());
  for (size_t c = 0; c < children.size(); ++c) {
    for (int k = 0; k < n; ++k) {
      child_poses[(c * n + k) * 3] = children[c]->state.objects[k].pose.x;
      child_poses[(c * n + k) * 3 + 1] = children[c]->state.objects[k].pose.y;
      child_poses[(c * n + k) * 3 + 2] = children[c]->state.objects[k].pose.theta;
    }
    meta[c * 3] = children[c]->depth;
    meta[c * 3 + 1] = children[c]->graspable_flag ? 1 : 0;
    meta[c * 3 + 2] = children[c]->dead_flag ? 1 : 0;
    rewards[c] = r[c];
  }
  *depth_cap = tree.tree_depth + tree.rollout_depth;
  return static_cast<int>(children.size());
}

// batch_simulate (pmbs.cpp:207-234) with WorkerPool(threads) on explicit new
// nodes: state i of the handle with node_meta[i] = {depth, graspable, dead};
// the tree's d_T / d_s are set so that d_T + d_s == depth_cap.  Times the
// reference call alone (bench.py's rollout CPU baseline).
int ref_batch_simulate(void* h, const int32_t* node_meta, int n_nodes, const ppg_params* p, uint64_t iteration,
                       int depth_cap, int threads, double* rewards, double* seconds) {
  States* st = static_cast<States*>(h);
  if (static_cast<int>(st->v.size()) < n_nodes) return -1;
  pmbs::ParallelConfig cfg = to_cfg(p);
  mcts::SearchTree tree;
  tree.tree_depth = depth_cap;
  tree.rollout_depth = 0;
  std::vector<std::unique_ptr<mcts::TreeNode>> own;
  std::vector<mcts::TreeNode*> nodes;
  for (int i = 0; i < n_nodes; ++i) {
    auto x = std::make_unique<mcts::TreeNode>();
    x->state = st->v[i];
    x->depth = node_meta[i * 3];
    x->graspable_flag = node_meta[i * 3 + 1] != 0;
    x->dead_flag = node_meta[i * 3 + 2] != 0;
    nodes.push_back(x.get());
    own.push_back(std::move(x));
  }
  std::unique_ptr<WorkerPool> pool;
  if (threads > 1) pool = std::make_unique<WorkerPool>(threads);
  const auto t0 = std::chrono::steady_clock::now();
  const auto r = pmbs::batch_simulate(tree, nodes, cfg, pool.get(), iteration);
  const auto t1 = std::chrono::steady_clock::now();
  if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
  for (int i = 0; i < n_nodes; ++i) rewards[i] = r[i];
  return 0;
}

// run_episode (bench.cpp:54-126) with the reference planner; returns actions
// used, sets completed and planning seconds.
int ref_run_episode(void* h, int i, const char* case_id, int trial, const ppg_params* p,
                    int threads, uint64_t seed_base, int action_cap, int32_t* completed,
                    double* planning_s, const char* log_path) {
  const WorldState& w = static_cast<States*>(h)->v.at(i);
  bench::BenchmarkConfig cfg;
  cfg.search = to_cfg(p);
  cfg.search.worker_threads = threads;
  cfg.action_cap = action_cap;
  cfg.seed_base = seed_base;
  const uint64_t seed = bench::episode_seed(seed_base, case_id, trial);
  std::ofstream log_file;
  if (log_path && log_path[0]) log_file.open(log_path);
  const bench::EpisodeResult r =
      bench::run_episode(w, case_id, trial, cfg, seed, log_file.is_open() ? &log_file : nullptr);
  *completed = r.completed ? 1 : 0;
  *planning_s = r.planning_time_s;
  return r.actions_used;
}

// bench::replay_log (bench.cpp:319-377): 1 when the JSONL episode log's
// recorded actions re-fold through the reference simulator with matching
// state digests.
int ref_replay_log(const char* path, char* report, int cap) {
  std::ostringstream out;
  const bool ok = bench::replay_log(path, out);
  const std::string s = out.str();
  if (report && cap > 0) {
    const size_t m = std::min<size_t>(s.size(), static_cast<size_t>(cap - 1));
    std::memcpy(report, s.data(), m);
    report[m] = '\0';
  }
  return ok ? 1 : 0;
}

}  // extern "C"
