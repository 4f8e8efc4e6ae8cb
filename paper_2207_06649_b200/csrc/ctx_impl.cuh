// ctx_impl.cuh — internals shared by the C-ABI translation units (ctx.cu,
// dtree.cu): kernel declarations, the context struct, device buffers and the
// launch helpers.  Not part of the public ABI.
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "ctx.h"
#include "kernels.cuh"

namespace ppg {

template <bool kCount>
__global__ void resolve_kernel(const __grid_constant__ SimConst C, ResolveArgs a);
__global__ void shape_prep_kernel(ShapesDev S, const int* kind, const double* radius, const int* nv,
                                  const double* verts, const int* target);
__global__ void sample_kernel(const __grid_constant__ SimConst C, SampleArgs a);
__global__ void grasp_kernel(const __grid_constant__ SimConst C, SampleArgs a);
__global__ void expand_kernel(const __grid_constant__ SimConst C, ExpandArgs a);
__global__ void lock_init_kernel(const __grid_constant__ SimConst C, LockArgs a);
__global__ void lock_harvest_kernel(const __grid_constant__ SimConst C, LockArgs a);
__global__ void lock_harvest_local_kernel(const __grid_constant__ SimConst C, LockArgs a);
__global__ void lock_harvest_apply_kernel(const __grid_constant__ SimConst C, LockArgs a);
__global__ void lock_step_kernel(const __grid_constant__ SimConst C, LockArgs a);
__global__ void lock_step_count_kernel(const __grid_constant__ SimConst C, LockArgs a, unsigned long long* ops);
__global__ void lock_sample_kernel(const __grid_constant__ SimConst C, LockArgs a);
__global__ void expand_post_kernel(const __grid_constant__ SimConst C, ExpandArgs a);
__global__ void poly_order_key_kernel(ResolveArgs a, unsigned* key, int* val);
template <bool kPoly>
__global__ void sample_grasp_warp_kernel(const __grid_constant__ SimConst C, SampleArgs a);
template <bool kPoly>
__global__ void expand_post_warp_kernel(const __grid_constant__ SimConst C, ExpandArgs a);
template <int NW, bool kPoly>
__global__ void resolve_warp_kernel(const __grid_constant__ SimConst C, ResolveArgs a);
template <int NW, bool kPoly>
__global__ void expand_warp_kernel(const __grid_constant__ SimConst C, ExpandArgs a);
template <int NW, bool kPoly>
__global__ void lock_step_warp_kernel(const __grid_constant__ SimConst C, LockArgs a);
constexpr int kWarpMaxN = 23;
constexpr int kPolyMaxN = 16;  // warp_poly.cuh
constexpr int kChunks = 4;     // slices of a pipelined host-buffer batch_resolve
constexpr int kMaxSlices = 32; // slices of a streamed host-buffer batch_resolve
constexpr int kWarpsPerBlock = 4;
// pair-mask words of the latency-mode kernels (warp_env.cuh warp_words_for)
constexpr int warp_words(int n) { return n <= 8 ? 1 : n <= 11 ? 2 : n <= 16 ? 4 : 8; }
// Launches KERNEL<NW, poly> (one warp per item, `items` items) for n objects;
// poly: the scene has polygons (warp_poly.cuh, n <= kPolyMaxN).
#define PPG_WARP_LAUNCH(KERNEL, poly, n, items, st, ...)                                    \
  do {                                                                                      \
    const int g_ = ((items) + kWarpsPerBlock - 1) / kWarpsPerBlock;                         \
    const int w_ = warp_words(n);                                                           \
    if (poly) {                                                                             \
      if (w_ == 1) KERNEL<1, true><<<g_, kWarpsPerBlock * 32, 0, st>>>(__VA_ARGS__);        \
      else if (w_ == 2) KERNEL<2, true><<<g_, kWarpsPerBlock * 32, 0, st>>>(__VA_ARGS__);   \
      else KERNEL<4, true><<<g_, kWarpsPerBlock * 32, 0, st>>>(__VA_ARGS__);                \
    } else if (w_ == 1) {                                                                   \
      KERNEL<1, false><<<g_, kWarpsPerBlock * 32, 0, st>>>(__VA_ARGS__);                    \
    } else if (w_ == 2) {                                                                   \
      KERNEL<2, false><<<g_, kWarpsPerBlock * 32, 0, st>>>(__VA_ARGS__);                    \
    } else if (w_ == 4) {                                                                   \
      KERNEL<4, false><<<g_, kWarpsPerBlock * 32, 0, st>>>(__VA_ARGS__);                    \
    } else {                                                                                \
      KERNEL<8, false><<<g_, kWarpsPerBlock * 32, 0, st>>>(__VA_ARGS__);                    \
    }                                                                                       \
  } while (0)
__global__ void lock_post_kernel(const __grid_constant__ SimConst C, LockArgs a);
__global__ void lock_async_init_kernel(const __grid_constant__ SimConst C, LockArgs a);
__global__ void wave_harvest_kernel(const __grid_constant__ SimConst C, LockArgs a);
__global__ void wave_pack_kernel(LockArgs a);
__global__ void wave_pack_pending_kernel(LockArgs a);
__global__ void wave_sample_kernel(const __grid_constant__ SimConst C, LockArgs a);
__global__ void wave_post_kernel(const __grid_constant__ SimConst C, LockArgs a);
template <int NW, bool kPoly, bool kSpecul>
__global__ void lock_async_kernel(const __grid_constant__ SimConst C, LockArgs a);
__global__ void lock_sample_warp_kernel(const __grid_constant__ SimConst C, LockArgs a);
__global__ void lock_post_warp_kernel(const __grid_constant__ SimConst C, LockArgs a);
__global__ void lock_report_kernel(const __grid_constant__ SimConst C, LockArgs a);
__global__ void lock_repurpose_kernel(const __grid_constant__ SimConst C, LockArgs a, const int32_t* env,
                                      const int32_t* node, int count);
__global__ void fp64_peak_kernel(double* out, int iters, double b, double c);
__global__ void debug_sincos_kernel(const double* x, int n, double* s, double* c);
template <int NMAX, bool kFix>
__global__ void resolve_disc_kernel(const __grid_constant__ SimConst C, ResolveArgs a, int* next_env);

constexpr int kBlock = 128;
constexpr int kDiscBlock = 128;  // resolve_disc.cu kDB
constexpr int kNumDisc = 10;
constexpr int kDiscSizes[kNumDisc] = {4, 6, 8, 10, 11, 12, 14, 16, 18, 20};
constexpr int kDiscMaxN = 20;  // the lane-per-env disc kernel's largest object count
constexpr size_t kMaxSmem = kPosePlanes * kMaxObjects * kBlock * sizeof(double);

}  // namespace ppg

using namespace ppg;

#define CK(call)                                                                         \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess) {                                                             \
      ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);                     \
      return PPG_ECUDA;                                                                  \
    }                                                                                    \
  } while (0)

namespace ppg {

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    size_t want = bytes < 256 ? 256 : bytes;
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) cap = want;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

}  // namespace ppg

namespace ppg {
struct DTreeState;
void dtree_release(ppg_ctx* ctx);
struct Group;  // multi.cu: the shards of a multi-GPU context and their exchange
}  // namespace ppg

struct ppg_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  ppg_params params{};
  std::string err;
  // shared scene (ppg_set_scene)
  bool has_scene = false;
  bool scene_all_discs = false;
  ShapesDev scene;
  std::vector<int32_t> h_kind, h_nv, h_target;
  std::vector<double> h_radius, h_verts;
  double side = 0.288, margin = 0.0;
  DevBuf scene_buf, scene_in;
  // per-call shape tables (batch_resolve with per-env shapes)
  DevBuf shape_buf, shape_in;
  // I/O scratch
  DevBuf b_in, b_push, b_out, b_status, b_resid, b_a, b_b, b_c, b_d, b_e;
  // lockstep state
  DevBuf l_node, l_pushes, l_done, l_byg, l_harv, l_flag, l_reward, l_poses, l_mt, l_mtidx;
  DevBuf l_W, l_rew, l_active, l_nactive, l_counters, l_npose, l_nmeta;
  DevBuf b_counter;              // persistent-kernel work counter
  DevBuf l_push, l_status, l_stepping, l_rec;
  LockArgs la{};        // current lockstep session
  ResolveArgs lra{};    // its in-place physics arguments
  SimConst lc{};        // its constants
  int lock_active_hint = 0;
  ppg_simulate_fn sim_hook = nullptr;
  void* sim_hook_user = nullptr;
  int32_t* h_nactive = nullptr;  // pinned
  int num_sms = 148;
  int disc_blocks_per_sm[kNumDisc] = {};  // resolve_disc_kernel<kDiscSizes[k]>
  bool disc_kernels = false;
  bool force_generic = false;             // PPG_FORCE_GENERIC=1: A/B the generic kernel
  int disc_bps_override = 0;              // PPG_DISC_BLOCKS_PER_SM: cap resident blocks (experiments)
  // pipelined batch_resolve (host buffers): per-slice streams and shape tables
  cudaStream_t chunk_stream[ppg::kChunks] = {};
  cudaEvent_t chunk_ev[ppg::kChunks] = {};  // slice k's host->device copies done
  DevBuf chunk_in[ppg::kChunks], chunk_buf[ppg::kChunks];
  DevBuf ord_buf[ppg::kChunks];          // polygon batches: launch-order keys, env order, sort scratch
  ppg::DTreeState* dtree = nullptr;       // device-resident PMBS tree (dtree.cu)
  int planner = 0;                        // PPG_PLANNER_AUTO / _HOST / _DEVICE (PPG_PLANNER env)
  int warp_max_envs = 2048;             // batch_resolve on discs (n <= kDiscMaxN): latency mode up to this many envs; PPG_WARP_MAX
  int hybrid_min_envs = 8192;            // lockstep rounds with >= this many active envs (discs, n <= kDiscMaxN)
                                          // run the hybrid warp-sampler / lane-physics round; PPG_HYBRID_MIN
  bool warp_max_explicit = false;        // PPG_WARP_MAX given: a hard cap for every scene type
  bool warp_poly = true;                  // polygon scenes in latency mode; PPG_WARP_POLY=0 disables
  // streamed batch_resolve (host buffers, disc batches): ONE physics launch
  // overlapping the slice copies; stream memory operations (driver API)
  // signal "slice k resident" to the kernel and "slice k finished" to the
  // copy-back stream
  ppg::DevBuf b_pipe;                    // ready flags [kMaxSlices] | done counters [kMaxSlices]
  unsigned* h_epochs = nullptr;          // pinned [kMaxSlices]: ready-flag values copied by the copy-in stream
  unsigned pipe_epoch = 0;
  int streamed = -1;                      // -1 not probed, 0 off (PPG_STREAMED=0 / no stream mem ops), 1 on
  void* fn_write32 = nullptr;             // cuStreamWriteValue32
  void* fn_wait32 = nullptr;              // cuStreamWaitValue32
  cudaStream_t pipe_stream[3] = {};       // host->device copies, physics, device->host copies
  cudaEvent_t pipe_ev = nullptr;          // slice 0 resident
  // multi-GPU (multi.cu): a rank context (ppg_create_rank, one process per
  // GPU) or a multi-device context (ppg_create_multi, one process) points at
  // its group; batch_simulate / run_pmbs then shard the rollout batch
  ppg::Group* group = nullptr;
  ppg::DevBuf l_go;                       // sharded harvest: "any env active" (device int)
  ppg::DevBuf trace_buf;                  // PPG_STEP_TRACE: per-step records (experiments)
  ppg::DevBuf l_around, l_astate, l_aW, l_actr, l_adl, l_actl;  // asynchronous lockstep state
  int async_mode = -1;                    // -1 not read, 0 off (PPG_ASYNC=0), 1 on
  int wave_mode = -1;                     // -1 not read, 0 off (PPG_WAVE=0), 1 on
  int wave_budget = 160;                  // projection iterations per env per wave (PPG_WAVE_BUDGET)
  int wave_switch = 12288;                // envs still running below which waves hand over to async (PPG_WAVE_SWITCH)
  ppg::DevBuf l_fin, l_rsi, l_ract;       // wave rounds: post list, resumable physics progress
  ppg::DevBuf l_gring;                   // sharded wave rounds: the exchanged ring (LockArgs.g_ring)
  ppg::DevBuf l_aP;                      // asynchronous lockstep: pending bounds ring (LockArgs.a_P)
  ppg::DevBuf l_spec;                    // asynchronous lockstep: held speculative steps (LockArgs.a_spec)
  int32_t* h_go = nullptr;                // pinned copy
};

SimConst make_const(const ppg_params& p, int n, double side, double margin);
size_t disc_smem(int nmax);
size_t smem_for(int n);
// fixpoint: the variant that ends a substep at a bit-identical fixed point
// (jammed pushes, frequent in rollouts); batch_resolve uses the plain one
int launch_disc(ppg_ctx* ctx, const SimConst& C, const ResolveArgs& a, int n, int work, cudaStream_t st,
                bool zero_counter = true, int slot_counter = 0, bool fixpoint = true);
bool use_disc(const ppg_ctx* ctx, bool all_discs, int n);
bool use_warp(const ppg_ctx* ctx, bool all_discs, int n, int envs, bool pmbs);
enum class RoundMode { kWarp, kHybrid, kLaneDisc, kGeneric, kAdaptive };
RoundMode round_mode(const ppg_ctx* ctx, int n, int envs);
int lock_round_on(ppg_ctx* ctx, const SimConst& C, const LockArgs& a, const ResolveArgs& ra, int work,
                  RoundMode mode, cudaStream_t st);
// Asynchronous lockstep (warp_env.cu lock_async_kernel): runs every remaining
// round of the current lockstep call; `work` = the most envs it may own.
// PPG_ASYNC=0 disables it (lockstep rounds everywhere).
bool async_enabled(const ppg_ctx* ctx);
int launch_async(ppg_ctx* ctx, const SimConst& C, const LockArgs& a, int work, cudaStream_t st, bool cont);
// Wave rounds (warp_env.cu wave_*_kernel): one wave = harvest, sample,
// budgeted lane physics, post.  PPG_WAVE=0 disables them (barrier hybrid rounds).
bool wave_enabled(const ppg_ctx* ctx);
bool speculate_enabled();  // PPG_SPECULATE=0 switches speculative re-purposing off
// speculation pays where envs wait on decisions (small batches); wide batches
// measured ~1 % slower with it (profiles/r2g_speculation_ab.txt)
constexpr int kSpecMaxEnvs = 2048;
int launch_wave(ppg_ctx* ctx, const SimConst& C, const LockArgs& a, const ResolveArgs& ra, int work, cudaStream_t st);
int lock_setup(ppg_ctx* ctx, const double* node_poses, const int32_t* node_meta, int n_nodes, int used,
               int used_global, int env_lo, int leaf_parallel, uint64_t seed, uint64_t iteration, int depth_cap);
int lock_round(ppg_ctx* ctx, int act);
int lock_check(ppg_ctx* ctx, int n_nodes, int n_envs, int depth_cap);
unsigned long long* step_trace_buffer(ppg_ctx* ctx);  // PPG_STEP_TRACE set: the record buffer, else null
void step_trace_dump(ppg_ctx* ctx);                   // appends the records to $PPG_STEP_TRACE

namespace ppg {
// multi.cu: the shards of a multi-GPU context.  Member k of this process is
// global shard rank0 + k of `world`; members all run the same calls (SPMD).
struct Group;
int group_size(const Group* g);
ppg_ctx* group_member(const Group* g, int k);
int group_rank0(const Group* g);
int group_world(const Group* g);
// In-place exchange over every shard (all ranks): sum of int32 / max of
// uint64 (bit patterns of non-negative doubles), enqueued on each member's
// stream; bufs[k] belongs to member k.
int group_allreduce_sum_i32(ppg_ctx* ectx, Group* g, int32_t* const* bufs, size_t count);
int group_allreduce_max_u64(ppg_ctx* ectx, Group* g, unsigned long long* const* bufs, size_t count);
int group_allreduce_sum_i64(ppg_ctx* ectx, Group* g, long long* const* bufs, size_t count);
// Waits for every member's stream (bounded by PPG_NCCL_TIMEOUT_S; a timeout
// aborts the communicators and reports an error instead of hanging).
int group_wait(ppg_ctx* ectx, Group* g);
// Sharded wave rounds: after the round-0 harvest, every remaining round as
// waves with ONE exchange per wave (multi.cu).  Member k runs la[k] / ra[k]
// with constants C[k]; P = n_nodes of the call; work = grid sizing.
struct ShardWave {
  ppg_ctx* c;
  const SimConst* C;
  LockArgs la;
  ResolveArgs ra;
};
bool shard_waves_enabled(const ppg_ctx* ctx);
int sharded_wave_rounds(ppg_ctx* ectx, Group* g, std::vector<ShardWave>& sw, int P, int work);
void group_destroy(ppg_ctx* ctx);
int simulate_sharded(ppg_ctx* ctx, const double* node_poses, const int32_t* node_meta, int n_nodes, int n_envs,
                     int leaf_parallel, uint64_t seed, uint64_t iteration, int depth_cap, double* rewards_out,
                     int64_t* counters);
int run_pmbs_sharded(ppg_ctx* ctx, const double* root_poses, double* action_out, ppg_search_stats* stats,
                     char* sig_buf, int64_t sig_cap, int64_t* sig_len);
}  // namespace ppg

// internal (not in include/pushplan_gpu.h): the search root's sample_pushes +
// graspable in one launch (ctx.cu), used by run_pmbs's setup (dtree.cu)
extern "C" int ppg_root_sample_grasp(ppg_ctx* ctx, const double* poses, double* untried, int32_t* count,
                                     uint8_t* graspable, const double** untried_dev);
