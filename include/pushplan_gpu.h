/*
 * pushplan_gpu.h — C-ABI of the B200-native PMBS batched-rollout hot path.
 *
 * This is the drop-in boundary: plain pointers and sizes, int return codes, no
 * exceptions and no torch types.  Each entry point names the reference
 * interface (arxiv 2207.06649 "pushplan", /root/reference/proj/core) that it
 * replaces.  A host binding (C++ adapter, ctypes, ...) marshals the reference
 * value types into the flat arrays below; see INTEGRATION.md.
 *
 * Array conventions (all host pointers unless a function name ends in _dev):
 *   poses     [E][n][3]  double  (x, y, theta) per object, reference Pose
 *                               (world.hpp:49-56)
 *   pushes    [E][4]     double  (x_s, y_s, x_e, y_e), reference PushAction
 *                               (world.hpp:79-85)
 *   status    [E]        int32   PPG_OK / PPG_START_COLLISION / PPG_NOT_CONVERGED
 *                               (the two SimError throw sites push_sim.cpp:60-62
 *                               and :123-128)
 *   shapes    one table per environment or one table shared by all, see
 *             ppg_shapes (reference ObjectShape world.hpp:33-46).
 */
#ifndef PUSHPLAN_GPU_H_
#define PUSHPLAN_GPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PPG_MAX_OBJECTS 32
#define PPG_MAX_VERTICES 8

/* return codes */
#define PPG_SUCCESS 0
#define PPG_EINVAL -1       /* bad argument (reference: SimError / SearchError on size checks) */
#define PPG_ECUDA -2        /* CUDA runtime failure */
#define PPG_ENOLEGAL -3     /* root has no legal push (reference SearchError mcts.cpp:244, pmbs.cpp:248) */
#define PPG_ENODEVICE -4    /* no CUDA device: the product has no CPU fallback */

/* per-element status (reference PushResult.error, push_sim.hpp:38-43) */
#define PPG_OK 0
#define PPG_START_COLLISION 1  /* push_sim.cpp:60-62 */
#define PPG_NOT_CONVERGED 2    /* push_sim.cpp:123-128 */

/* object kinds (reference ObjectShape::Kind, world.hpp:34) */
#define PPG_DISC 0
#define PPG_POLYGON 1

/* Scene shapes.  n_tables == 1: every environment shares the table (a PMBS
 * search: only poses differ between tree nodes); n_tables == E: one table per
 * environment (reference batch_resolve over arbitrary WorldStates). */
typedef struct ppg_shapes {
  int32_t n_objects;            /* objects per environment, 1..PPG_MAX_OBJECTS */
  int32_t n_tables;             /* 1 or E */
  const int32_t* kind;          /* [n_tables][n_objects] PPG_DISC / PPG_POLYGON */
  const double* radius;         /* [n_tables][n_objects] disc radius */
  const int32_t* n_vertices;    /* [n_tables][n_objects]; NULL when all discs */
  const double* vertices;       /* [n_tables][n_objects][PPG_MAX_VERTICES][2] local CCW; NULL when all discs */
  const int32_t* target_index;  /* [n_tables] (WorldState::target_index, world.hpp:66) */
  double side_length;           /* Workspace::side_length (world.hpp:18) */
  double boundary_margin;       /* Workspace::boundary_margin (world.hpp:19) */
} ppg_shapes;

/* Every knob of the reference config structs, flattened.  ppg_params_default
 * fills the reference defaults. */
typedef struct ppg_params {
  /* GripperTip (world.hpp:86-89) */
  double tip_radius;            /* 0.012 */
  double tip_clearance;         /* 0.002 */
  /* SimParams (push_sim.hpp:14-20) */
  double push_distance;         /* 0.05 */
  int32_t substeps;             /* 64 */
  int32_t max_projection_iters; /* 32 */
  double eps_pen;               /* 1e-4 */
  double rotation_gain;         /* 1.0 */
  /* GraspGeometry (actions.hpp:21-26) */
  double finger_width;          /* 0.02 */
  double finger_thickness;      /* 0.01 */
  double opening;               /* 0.085 */
  double approach_clearance;    /* 0.003 */
  /* SearchConfig (mcts.hpp:30-44) */
  double gamma;                 /* 0.8 */
  double c_explore;             /* 0.3 */
  int32_t tree_depth;           /* 7 */
  int32_t rollout_depth;        /* 3 */
  int32_t pushes_per_object;    /* 16 */
  double margin_threshold;      /* 0.003 */
  uint64_t rng_seed;            /* 0 */
  int32_t rank_by_ucb;          /* 0 */
  int32_t budget_iterations;    /* 1: Budget::iterations(max_iterations); 0: Budget::seconds(max_seconds) */
  int64_t max_iterations;       /* 0 */
  double max_seconds;           /* 60.0 */
  /* ParallelConfig (pmbs.hpp:24-28) */
  int32_t n_envs;               /* 64 */
  int32_t leaf_parallel;        /* 1 */
} ppg_params;

typedef struct ppg_ctx ppg_ctx;

/* Search statistics (reference SearchStats, mcts.hpp:80-85). */
typedef struct ppg_search_stats {
  int64_t iterations;
  int64_t expansions;
  double elapsed_s;
  int32_t stop_reason;          /* 0 budget, 1 explored, 2 early_stop */
  int32_t final_tree_depth;     /* SearchTree::tree_depth at return */
  int64_t env_steps;            /* resolve_push calls: expansions + rollout steps */
  int64_t rollout_steps;        /* RolloutCursor::step calls that ran a push */
  int64_t lockstep_rounds;
  uint64_t signature_fnv;       /* FNV-1a-64 of tree_signature() text (mcts.cpp:296-300) */
  int64_t n_nodes;
  double select_s;              /* host time in select_batch + reset_virtual */
  double expand_s;              /* batch_expand: device prepare + host attach */
  double simulate_s;            /* batch_simulate on the device */
  double backprop_s;            /* host backprop + early-stop bookkeeping */
} ppg_search_stats;

/* Fills the reference defaults. */
void ppg_params_default(ppg_params* p);

/* Version / build string, e.g. "pmbs_b200 sm_100a fmad=false". */
const char* ppg_version(void);

/* Number of visible CUDA devices (0 on a host without a GPU; never touches a
 * kernel). */
int ppg_device_count(void);

/* Creates a context on `device` (the WorkerPool seam of the reference:
 * pmbs.cpp:250-251, push_sim.cpp:146-150).  Returns NULL and sets *err on
 * failure.  One context per host thread. */
ppg_ctx* ppg_create(int device, const ppg_params* params, int* err);
void ppg_destroy(ppg_ctx* ctx);
const char* ppg_last_error(ppg_ctx* ctx);

/* Replaces the context's parameters (takes effect on the next call). */
int ppg_set_params(ppg_ctx* ctx, const ppg_params* params);

/* Installs the shared scene shapes used by ppg_expand / ppg_simulate /
 * ppg_run_pmbs (SearchTree::create, mcts.cpp:28-39, fixes the shapes of a
 * search).  shapes->n_tables must be 1. */
int ppg_set_scene(ppg_ctx* ctx, const ppg_shapes* shapes);

/* batch_resolve (push_sim.hpp:48-51, push_sim.cpp:132-152): element-wise
 * resolve_push (push_sim.cpp:58-130) with per-element status; never aborts
 * siblings.  residual[e] = final max pairwise penetration (NULL allowed).
 * shapes == NULL uses the context scene.  Synchronous w.r.t. host buffers.
 * All-disc batches of >= 32K envs with per-env shapes are streamed (the
 * copies overlap one physics launch); when poses_out / status / residual are
 * pinned host memory (cudaHostAlloc, pinned torch tensors) the kernel writes
 * the results into them directly.  Pageable buffers work too (copy-back). */
int ppg_batch_resolve(ppg_ctx* ctx, const ppg_shapes* shapes, const double* poses_in,
                      const double* pushes, int E, double* poses_out, int32_t* status,
                      double* residual);

/* Same on device-resident buffers (all pointers are device pointers; shape
 * arrays too), enqueued on `stream` (a cudaStream_t, NULL = default stream),
 * asynchronous. */
int ppg_batch_resolve_dev(ppg_ctx* ctx, const ppg_shapes* shapes_dev, const double* poses_in,
                          const double* pushes, int E, double* poses_out, int32_t* status,
                          double* residual, void* stream);

/* sample_pushes (actions.hpp:39-40, actions.cpp:51-73) for E states:
 * out[e][k] for k < count[e] in (object, angle) order, capacity n_objects *
 * pushes_per_object per state.  shapes == NULL uses the context scene. */
int ppg_sample_pushes(ppg_ctx* ctx, const ppg_shapes* shapes, const double* poses, int E, double* out,
                      int32_t* count);

/* graspable (actions.hpp:47-48, actions.cpp:113-147) for E states sharing the
 * context scene: flag, margin, best (x, y, angle_index; angle_index -1 when no
 * feasible pose). */
int ppg_graspable(ppg_ctx* ctx, const double* poses, int E, uint8_t* graspable,
                  double* margin, double* best_x, double* best_y, int32_t* best_angle);

/* batch_expand prepare step (pmbs.hpp:51-52, pmbs.cpp:82-93): per pair,
 * resolve_push -> sample_pushes (full list) -> graspable.  child_poses and
 * untried follow the conventions above; untried capacity per pair is
 * n_objects * pushes_per_object. */
int ppg_expand(ppg_ctx* ctx, const double* parent_poses, const double* actions, int P,
               double* child_poses, int32_t* status, uint8_t* graspable, int32_t* n_untried,
               double* untried);

/* batch_simulate / lockstep_simulate (pmbs.hpp:73-82, pmbs.cpp:133-234): the
 * leaf-parallel lockstep rollouts of n_envs environments over n_nodes new
 * nodes; env e uses the MT19937-64 stream keyed (seed, iteration, e)
 * (rng.hpp:21-23).  node_meta[i] = {depth, graspable, dead}.  depth_cap =
 * tree_depth + rollout_depth as they stand after this iteration's expansion
 * (pmbs.cpp:230-231).  rewards_out[i] = max over node i's rollouts.
 * counters (optional, 4 x int64): rollout steps, rounds, re-purposes, resolve
 * calls. */
int ppg_simulate(ppg_ctx* ctx, const double* node_poses, const int32_t* node_meta, int n_nodes,
                 int n_envs, int leaf_parallel, uint64_t seed, uint64_t iteration, int depth_cap,
                 double* rewards_out, int64_t* counters);

/* ppg_simulate's algorithmic work (the rollout roofline numerator, SURVEY
 * 8d): the same lockstep (bit-identical rollouts) through an instrumented
 * one-lane step kernel; ops_out[3] = FP64 ops (+,-,*,/,sqrt = 1 each) of the
 * resolve_push, sample_pushes and graspable calls of every rollout step. */
int ppg_simulate_count(ppg_ctx* ctx, const double* node_poses, const int32_t* node_meta, int n_nodes, int n_envs,
                       int leaf_parallel, uint64_t seed, uint64_t iteration, int depth_cap, int64_t* ops_out,
                       int64_t* counters);

/* ---- multi-GPU contexts (BASELINE configs[4]) ----
 * The rollout batch of every PMBS iteration (batch_simulate, pmbs.cpp:207-234)
 * is sharded by environment over G GPUs: shard r owns a contiguous range of
 * the global env batch (RNG keys and the env -> node split stay global), the
 * search tree is replicated, and each lockstep round exchanges ONE vector —
 * the per-node remaining work W (pmbs.cpp:157-163), all-reduced (sum) over
 * NVLink — so every shard re-purposes its own finished envs to the same
 * argmax node as the reference's sequential harvest (pmbs.cpp:165-187).
 * Disc scenes run the rounds as waves: one all-reduce per wave of the ring
 * of per-round W vectors and (arrived, gone) counts, from which every shard
 * takes the same (early) decisions.
 * Per-node rewards are all-reduced (max) once per iteration.  Results
 * (decision, tree, rewards) are bit-identical for every G.  ppg_simulate and
 * ppg_run_pmbs* on such a context run sharded; every other call runs on the
 * context's own device.  All ranks / shards must make the same calls (SPMD).
 *
 * ppg_create_rank: one process per GPU (torchrun); rank 0 makes the NCCL id
 * with ppg_nccl_unique_id and the caller broadcasts it (128 bytes).
 * ppg_create_multi: one process driving n_dev GPUs (ncclCommInitAll);
 * flags PPG_MULTI_EMULATE: n_dev shards on ONE device (devices all equal)
 * exchanging through a device kernel — the test double of the NCCL path on a
 * single GPU.  ppg_destroy on the returned context releases every shard. */
#define PPG_MULTI_EMULATE 1
int ppg_nccl_unique_id(uint8_t* id /* 128 bytes */);
ppg_ctx* ppg_create_rank(int device, int rank, int world, const uint8_t* nccl_id, const ppg_params* params,
                         int* err);
ppg_ctx* ppg_create_multi(const int* devices, int n_dev, int flags, const ppg_params* params, int* err);
/* rank = global shard index of this context's first shard; transport 0 none,
 * 1 NCCL, 2 emulated (one device). */
int ppg_shard_info(ppg_ctx* ctx, int* rank, int* world, int* shards_here, int* transport);

/* ---- sharded lockstep (multi-GPU batch_simulate) ----
 * The lockstep engine split by environment: this context owns global envs
 * [env_lo, env_hi) of a batch of used_envs (= n_envs with leaf parallelism,
 * else n_nodes).  env -> node split and RNG keys use GLOBAL env indices, so
 * the union of the shards reproduces the unsharded batch exactly.  A driver
 * (python: paper_2207_06649_b200.sharded) loops:
 *   report -> exchange records / W -> global harvest (identical on every
 *   rank) -> repurpose -> step,
 * until no rank has an active env.  ppg_lock_report returns this shard's
 * newly finished envs in increasing global index (env, node, by_grasp,
 * reward; capacity env_hi - env_lo) and its remaining-work vector
 * W_local[n_nodes] = sum over assigned not-done envs of cap - pushes
 * (pmbs.cpp:157-163). */
int ppg_lock_begin(ppg_ctx* ctx, const double* node_poses, const int32_t* node_meta, int n_nodes, int used_envs,
                   int env_lo, int env_hi, int leaf_parallel, uint64_t seed, uint64_t iteration, int depth_cap);
int ppg_lock_report(ppg_ctx* ctx, int32_t* rec_env, int32_t* rec_node, uint8_t* rec_grasp, double* rec_reward,
                    int32_t* n_rec, int32_t* w_local, int32_t* n_active);
int ppg_lock_repurpose(ppg_ctx* ctx, const int32_t* env, const int32_t* node, int count);
int ppg_lock_step(ppg_ctx* ctx);
/* counters (4 x int64): rollout steps, -, -, resolve calls of this shard */
int ppg_lock_counters(ppg_ctx* ctx, int64_t* counters);

/* Replaces the planner's batch_simulate (ppg_run_pmbs) with a caller
 * function of ppg_simulate's signature (minus ctx) — e.g. the sharded
 * multi-GPU driver.  fn == NULL restores the built-in device lockstep. */
typedef int (*ppg_simulate_fn)(void* user, const double* node_poses, const int32_t* node_meta, int n_nodes,
                               int n_envs, int leaf_parallel, uint64_t seed, uint64_t iteration, int depth_cap,
                               double* rewards_out, int64_t* counters);
int ppg_set_simulate_hook(ppg_ctx* ctx, ppg_simulate_fn fn, void* user);

/* Planner selection for ppg_run_pmbs (also env PPG_PLANNER=host|device):
 * AUTO = DEVICE = the device-resident tree (dtree.cu; with a simulate hook
 * installed — the sharded multi-GPU driver — each iteration runs its rollouts
 * through the hook between two graph launches); HOST = tree on the host
 * (planner.cpp). */
#define PPG_PLANNER_AUTO 0
#define PPG_PLANNER_HOST 1
#define PPG_PLANNER_DEVICE 2
int ppg_set_planner(ppg_ctx* ctx, int mode);

/* run_pmbs (pmbs.hpp:91, pmbs.cpp:242-292) on the context scene and poses:
 * the full PMBS planning decision, batched expansion and lockstep rollouts
 * on the device, the tree per ppg_set_planner.  action_out[4] = chosen push.
 * Returns PPG_ENOLEGAL when the root has no legal push. */
int ppg_run_pmbs(ppg_ctx* ctx, const double* root_poses, double* action_out,
                 ppg_search_stats* stats);

/* run_pmbs with the search tree resident on the device: batched UCT leaf
 * selection with virtual visits (pmbs.cpp:12-63), expansion + attach
 * (:70-131), lockstep rollouts (:133-234) and backprop (:236-240) are one
 * CUDA-graph launch per PMBS iteration.  Same results as the host tree;
 * writes the tree signature like ppg_run_pmbs_sig (sig_buf may be NULL). */
int ppg_run_pmbs_device(ppg_ctx* ctx, const double* root_poses, double* action_out,
                        ppg_search_stats* stats, char* sig_buf, int64_t sig_cap, int64_t* sig_len);

/* Same, and also writes the tree_signature text (mcts.cpp:284-300) into
 * sig_buf (NUL-terminated, truncated to sig_cap); *sig_len = full length. */
int ppg_run_pmbs_sig(ppg_ctx* ctx, const double* root_poses, double* action_out,
                     ppg_search_stats* stats, char* sig_buf, int64_t sig_cap, int64_t* sig_len);

/* The search tree of the context's last ppg_run_pmbs* decision (the device
 * tree), for SearchResult::tree (mcts.hpp:87-91, pmbs.hpp:91): nodes in
 * creation order (root 0; a node's children in insertion order = increasing
 * index), parent[N] (-1 at the root), depth[N], action[N][4] (the push that
 * produced the node; zeros at the root), visits[N], q_sum[N], flags[N]
 * (bit0 graspable, bit1 dead), poses[N][n][3], untried_count[N] (untried
 * actions not yet expanded) and untried[U][4] (those actions, concatenated in
 * node order); scal[4] = {tree_depth, rollout_depth, es_level, n_objects} at
 * return.  Pass NULL arrays to read *n_nodes / *n_untried first. */
int ppg_tree_export(ppg_ctx* ctx, int64_t* n_nodes, int64_t* n_untried, int32_t* parent, int32_t* depth,
                    double* action, int64_t* visits, double* q_sum, uint8_t* flags, double* poses,
                    int32_t* untried_count, double* untried, int32_t* scal);

/* FNV-1a state digest (world.cpp:166-191) of E states sharing `shapes`
 * (n_tables 1 or E): bit-exact state identity. Host-only helper. */
int ppg_state_digest(const ppg_shapes* shapes, const double* poses, int E, uint64_t* out);

/* Algorithmic FP64 work counters for ppg_batch_resolve (SURVEY 8d formula):
 * runs an instrumented variant of the physics kernel on device buffers and
 * writes per-env counts [E][8] = {T_b, T_n, H_t, P_b, P_n, H_p, S, P_final}. */
int ppg_batch_resolve_count_dev(ppg_ctx* ctx, const ppg_shapes* shapes_dev,
                                const double* poses_in, const double* pushes, int E,
                                int64_t* counts_dev, void* stream);

/* Test helper (acceptance criterion 3, acceptance.cpp:255-281): runs the
 * device select_batch (pmbs.cpp:52-63, the dt_select_kernel of every PMBS
 * iteration graph) on one explicit tree: nodes in pre-order, children in
 * insertion order; node x has n_children[x] children and n_untried[x]
 * untried actions, flags bit0 graspable / bit1 dead (TreeNode, mcts.hpp:45-66).
 * Writes the selected pairs (node, untried index) in draw order (*n_sel = 0:
 * TreeExhausted), the nodes' virtual visits after the batch and their sum
 * after reset_virtual (pmbs.cpp:65-68). */
int ppg_debug_select_batch(ppg_ctx* ctx, int n_nodes, const int32_t* parent, const int32_t* depth,
                           const int64_t* visits, const double* q_sum, const uint8_t* flags,
                           const int32_t* n_children, const int32_t* n_untried, int tree_depth, int n_envs,
                           double c_explore, int32_t* sel_node, int32_t* sel_untried, int32_t* n_sel,
                           int64_t* vv_out, int64_t* vsum_after_reset);

/* Test helper: the device port of glibc sincos (the reference's libm,
 * __sincos_fma) on n arguments |x| < 105414350; bit-identical to the host. */
int ppg_debug_sincos(ppg_ctx* ctx, const double* x, int n, double* s, double* c);

/* Measurement helper (not on the hot path): the FP64 CUDA-core pipe peak in
 * DFMA instructions per second, from a dependent-chain microbenchmark on the
 * context's device — the roofline denominator of the FP64 kernels. */
int ppg_measure_fp64_peak(ppg_ctx* ctx, double* dfma_per_s, double* seconds);

/* ---- host-side input generators (no device needed) ---- */

/* bench::generate_case / generate_case_motif (bench.cpp:234-317): one scene
 * per seed, bit-identical to the reference generator (same libstdc++
 * std::mt19937_64 and distributions, same glibc).  motif 0 random, 1 ring,
 * 2 wall.  Outputs are [count][n_objects] tables in the ppg_shapes layout
 * plus poses [count][n_objects][3]; ok[c] = 0 where the reference throws
 * (rejection sampling exhausted).  `threads` host threads split the seeds. */
int ppg_generate_cases(int motif, int n_objects, double polygon_fraction, const uint64_t* seeds, int count,
                       int32_t* kind, double* radius, int32_t* n_vertices, double* vertices, double* poses,
                       int32_t* target_index, int32_t* ok, int threads);

/* out[c] = std::uniform_int_distribution<size_t>(0, n[c]-1) applied once to
 * keyed_rng(seed, a[c], b[c]) (rng.hpp:21-23, mcts.cpp:151-152); a or b may
 * be NULL (0). */
int ppg_keyed_picks(uint64_t seed, const uint64_t* a, const uint64_t* b, const uint64_t* n, int count,
                    uint64_t* out);

#ifdef __cplusplus
}
#endif

#endif /* PUSHPLAN_GPU_H_ */
