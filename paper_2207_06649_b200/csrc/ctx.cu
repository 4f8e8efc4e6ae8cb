// ctx.cu — the C-ABI (include/pushplan_gpu.h) over the sm_100a kernels:
// context, device buffers, shape upload and the host loops that drive the
// kernels.  The PMBS tree planner that sits on top lives in planner.cpp.
#include <cuda.h>  // stream memory operation types (entry points resolved at run time)
#include <cuda_runtime.h>
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>
#include <chrono>
#include <thread>

#include "ctx.h"
#include "kernels.cuh"

#include "ctx_impl.cuh"

SimConst make_const(const ppg_params& p, int n, double side, double margin) {
  SimConst C;
  std::memset(&C, 0, sizeof C);
  C.tip_r = p.tip_radius;
  C.tip_clear = p.tip_clearance;
  C.push_distance = p.push_distance;
  C.substeps = p.substeps;
  C.max_iters = p.max_projection_iters;
  C.eps_pen = p.eps_pen;
  C.gain = p.rotation_gain;
  C.side = side;
  C.margin = margin;
  C.finger_width = p.finger_width;
  C.finger_thickness = p.finger_thickness;
  C.opening = p.opening;
  C.approach_clearance = p.approach_clearance;
  C.margin_threshold = p.margin_threshold;
  C.na = p.pushes_per_object;
  C.n = n;
  static const bool no_fix = [] {
    const char* v = std::getenv("PPG_NO_FIXPOINT");
    return v && v[0] == '1';
  }();
  C.fixpoint = no_fix ? 0 : 1;
  // Same expressions and the same glibc as the reference (actions.cpp:59-60,
  // :77-78; mcts.cpp:132 std::pow(double, int) == pow(double, double)).
  const int n_per_object = p.pushes_per_object;
  for (int k = 0; k < n_per_object && k < kMaxNa; ++k) {
    const double angle = 2.0 * M_PI * k / n_per_object;
    C.dir_cos[k] = std::cos(angle);
    C.dir_sin[k] = std::sin(angle);
  }
  for (int k = 0; k < kGraspAngles; ++k) {
    const double angle = 2.0 * M_PI * k / kGraspAngles;
    C.g_cos[k] = std::cos(angle);
    C.g_sin[k] = std::sin(angle);
  }
  for (int k = 0; k < kMaxGammaPow; ++k) C.gamma_pow[k] = std::pow(p.gamma, static_cast<double>(k));
  return C;
}

int check_params(ppg_ctx* ctx, const ppg_params& p) {
  if (p.pushes_per_object > kMaxNa) {
    ctx->err = "pushes_per_object > 32 is not supported by the device sampler";
    return PPG_EINVAL;
  }
  if (p.substeps < 1 || p.max_projection_iters < 0) {
    ctx->err = "substeps must be >= 1";
    return PPG_EINVAL;
  }
  if (p.tree_depth + p.rollout_depth >= kMaxGammaPow) {
    ctx->err = "tree_depth + rollout_depth too large";
    return PPG_EINVAL;
  }
  return PPG_SUCCESS;
}

// Uploads host shape arrays (ppg_shapes) and runs shape_prep_kernel into `S`.
int upload_shapes(ppg_ctx* ctx, const ppg_shapes* sh, bool device_ptrs, DevBuf& in, DevBuf& buf, ShapesDev& S,
                  cudaStream_t st) {
  const int n = sh->n_objects, T = sh->n_tables;
  if (n < 1 || n > kMaxObjects || T < 1) {
    ctx->err = "n_objects must be in [1, 32] and n_tables >= 1";
    return PPG_EINVAL;
  }
  const size_t tn = static_cast<size_t>(T) * n;
  const size_t vbytes = tn * kMaxV * 2 * sizeof(double);
  // layout of `buf`: kind | rad | br | nv | verts | target
  const size_t off_rad = ((tn * 4 + 15) / 16) * 16;
  const size_t off_br = off_rad + tn * 8;
  const size_t off_nv = off_br + tn * 8;
  const size_t off_v = off_nv + ((tn * 4 + 15) / 16) * 16;
  const size_t off_t = off_v + vbytes;
  CK(buf.ensure(off_t + T * 4 + 16));
  char* b = buf.as<char>();
  S.kind = reinterpret_cast<int*>(b);
  S.rad = reinterpret_cast<double*>(b + off_rad);
  S.br = reinterpret_cast<double*>(b + off_br);
  S.nv = reinterpret_cast<int*>(b + off_nv);
  S.verts = reinterpret_cast<double*>(b + off_v);
  S.target = reinterpret_cast<int*>(b + off_t);
  S.T = T;
  S.n = n;
  const int* kind = sh->kind;
  const double* radius = sh->radius;
  const int* nv = sh->n_vertices;
  const double* verts = sh->vertices;
  const int* target = sh->target_index;
  if (!device_ptrs) {
    // stage host arrays: kind | radius | nv | verts | target
    const size_t o_r = ((tn * 4 + 15) / 16) * 16, o_nv = o_r + tn * 8, o_v = o_nv + ((tn * 4 + 15) / 16) * 16,
                 o_t = o_v + vbytes;
    CK(in.ensure(o_t + T * 4 + 16));
    char* q = in.as<char>();
    CK(cudaMemcpyAsync(q, sh->kind, tn * 4, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(q + o_r, sh->radius, tn * 8, cudaMemcpyHostToDevice, st));
    if (sh->n_vertices) CK(cudaMemcpyAsync(q + o_nv, sh->n_vertices, tn * 4, cudaMemcpyHostToDevice, st));
    else CK(cudaMemsetAsync(q + o_nv, 0, tn * 4, st));
    if (sh->vertices) CK(cudaMemcpyAsync(q + o_v, sh->vertices, vbytes, cudaMemcpyHostToDevice, st));
    else CK(cudaMemsetAsync(q + o_v, 0, vbytes, st));
    CK(cudaMemcpyAsync(q + o_t, sh->target_index, T * 4, cudaMemcpyHostToDevice, st));
    kind = reinterpret_cast<int*>(q);
    radius = reinterpret_cast<double*>(q + o_r);
    nv = reinterpret_cast<int*>(q + o_nv);
    verts = reinterpret_cast<double*>(q + o_v);
    target = reinterpret_cast<int*>(q + o_t);
  }
  const int threads = 256;
  const int total = static_cast<int>(tn > static_cast<size_t>(T) ? tn : T);
  shape_prep_kernel<<<(total + threads - 1) / threads, threads, 0, st>>>(S, kind, radius, nv, verts, target);
  CK(cudaGetLastError());
  return PPG_SUCCESS;
}

bool host_all_discs(const ppg_shapes* sh) {
  if (!sh->n_vertices && !sh->vertices) return true;
  const size_t tn = static_cast<size_t>(sh->n_tables) * sh->n_objects;
  for (size_t i = 0; i < tn; ++i)
    if (sh->kind[i] != PPG_DISC) return false;
  return true;
}

template <class F>
bool for_each_disc_kernel(F&& f) {
#define PPG_DISC_FN(N, X) reinterpret_cast<const void*>(&resolve_disc_kernel<N, X>)
  const void* fns[2][kNumDisc] = {
      {PPG_DISC_FN(4, false), PPG_DISC_FN(6, false), PPG_DISC_FN(8, false), PPG_DISC_FN(10, false),
       PPG_DISC_FN(11, false), PPG_DISC_FN(12, false), PPG_DISC_FN(14, false), PPG_DISC_FN(16, false),
       PPG_DISC_FN(18, false), PPG_DISC_FN(20, false)},
      {PPG_DISC_FN(4, true), PPG_DISC_FN(6, true), PPG_DISC_FN(8, true), PPG_DISC_FN(10, true),
       PPG_DISC_FN(11, true), PPG_DISC_FN(12, true), PPG_DISC_FN(14, true), PPG_DISC_FN(16, true),
       PPG_DISC_FN(18, true), PPG_DISC_FN(20, true)}};
#undef PPG_DISC_FN
  for (int v = 1; v >= 0; --v)  // occupancy is taken from the last call: the plain variant
    for (int k = 0; k < kNumDisc; ++k)
      if (!f(k, fns[v][k])) return false;
  return true;
}

// resolve_disc_kernel: doubles x | y | r | theta (theta for nmax <= 14), floats xf | yf
size_t disc_smem(int nmax) {
  return (static_cast<size_t>(nmax <= 14 ? 4 : 3) * sizeof(double) + 2 * sizeof(float)) * nmax * kDiscBlock;
}

size_t smem_for(int n) { return static_cast<size_t>(kPosePlanes) * n * kBlock * sizeof(double); }

// ---------------------------------------------------------------------------

extern "C" {

void ppg_params_default(ppg_params* p) {
  std::memset(p, 0, sizeof *p);
  p->tip_radius = 0.012;
  p->tip_clearance = 0.002;
  p->push_distance = 0.05;
  p->substeps = 64;
  p->max_projection_iters = 32;
  p->eps_pen = 1e-4;
  p->rotation_gain = 1.0;
  p->finger_width = 0.02;
  p->finger_thickness = 0.01;
  p->opening = 0.085;
  p->approach_clearance = 0.003;
  p->gamma = 0.8;
  p->c_explore = 0.3;
  p->tree_depth = 7;
  p->rollout_depth = 3;
  p->pushes_per_object = 16;
  p->margin_threshold = 0.003;
  p->rng_seed = 0;
  p->rank_by_ucb = 0;
  p->budget_iterations = 0;
  p->max_iterations = 0;
  p->max_seconds = 60.0;
  p->n_envs = 64;
  p->leaf_parallel = 1;
}

#ifdef PPG_FMA_VARIANT
const char* ppg_version(void) { return "pmbs_b200 0.2 sm_100a fp64 fmad=true (FMA variant: tolerance, not bit-exact)"; }
#else
const char* ppg_version(void) { return "pmbs_b200 0.2 sm_100a fp64 fmad=false"; }
#endif

int ppg_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

ppg_ctx* ppg_create(int device, const ppg_params* params, int* err) {
  if (err) *err = PPG_SUCCESS;
  const int nd = ppg_device_count();
  if (nd <= 0 || device < 0 || device >= nd) {
    if (err) *err = PPG_ENODEVICE;
    return nullptr;
  }
  auto* ctx = new ppg_ctx;
  ctx->device = device;
  if (params) ctx->params = *params;
  else ppg_params_default(&ctx->params);
  if (check_params(ctx, ctx->params) != PPG_SUCCESS) {
    if (err) *err = PPG_EINVAL;
    delete ctx;
    return nullptr;
  }
  bool ok = cudaSetDevice(device) == cudaSuccess && cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) == cudaSuccess &&
            cudaMallocHost(&ctx->h_nactive, sizeof(int32_t)) == cudaSuccess;
  const int smem = static_cast<int>(kMaxSmem);
  ok = ok && cudaFuncSetAttribute(resolve_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) == cudaSuccess;
  ok = ok && cudaFuncSetAttribute(resolve_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) == cudaSuccess;
  ok = ok && cudaFuncSetAttribute(sample_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) == cudaSuccess;
  ok = ok && cudaFuncSetAttribute(grasp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) == cudaSuccess;
  ok = ok && cudaFuncSetAttribute(expand_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) == cudaSuccess;
  ok = ok && cudaFuncSetAttribute(lock_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) == cudaSuccess;
  ok = ok && cudaFuncSetAttribute(lock_step_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) == cudaSuccess;
  ok = ok && cudaFuncSetAttribute(lock_sample_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) == cudaSuccess;
  ok = ok && cudaFuncSetAttribute(expand_post_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) == cudaSuccess;
  ok = ok && cudaFuncSetAttribute(lock_post_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) == cudaSuccess;
  ok = ok && cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device) == cudaSuccess;
  ok = ok && for_each_disc_kernel([&](int k, const void* fn) {
    return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(disc_smem(kDiscSizes[k]))) == cudaSuccess &&
           cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctx->disc_blocks_per_sm[k], fn, kDiscBlock,
                                                         disc_smem(kDiscSizes[k])) == cudaSuccess &&
           ctx->disc_blocks_per_sm[k] > 0;
  });
  ctx->disc_kernels = ok;
  {
    const char* fg = std::getenv("PPG_FORCE_GENERIC");
    ctx->force_generic = fg && fg[0] == '1';
    const char* wm = std::getenv("PPG_WARP_MAX");
    if (wm) {
      ctx->warp_max_envs = std::atoi(wm);
      ctx->warp_max_explicit = true;
    }
    const char* hm = std::getenv("PPG_HYBRID_MIN");
    if (hm) ctx->hybrid_min_envs = std::atoi(hm);
    const char* wp = std::getenv("PPG_WARP_POLY");
    if (wp) ctx->warp_poly = wp[0] != '0';
    const char* pl = std::getenv("PPG_PLANNER");
    if (pl) ctx->planner = !std::strcmp(pl, "host") ? PPG_PLANNER_HOST : !std::strcmp(pl, "device") ? PPG_PLANNER_DEVICE : 0;
    const char* bo = std::getenv("PPG_DISC_BLOCKS_PER_SM");
    ctx->disc_bps_override = bo ? std::atoi(bo) : 0;
  }
  if (!ok) {
    cudaGetLastError();
    if (err) *err = PPG_ECUDA;
    ppg_destroy(ctx);
    return nullptr;
  }
  return ctx;
}

void ppg_destroy(ppg_ctx* ctx) {
  if (!ctx) return;
  if (ctx->group && ppg::group_member(ctx->group, 0) == ctx) ppg::group_destroy(ctx);  // also the other shards
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  DevBuf* bufs[] = {&ctx->scene_buf, &ctx->scene_in, &ctx->shape_buf, &ctx->shape_in, &ctx->b_in, &ctx->b_push,
                    &ctx->b_out, &ctx->b_status, &ctx->b_resid, &ctx->b_a, &ctx->b_b, &ctx->b_c, &ctx->b_d,
                    &ctx->b_e, &ctx->l_node, &ctx->l_pushes, &ctx->l_done, &ctx->l_byg, &ctx->l_harv,
                    &ctx->l_flag, &ctx->l_reward, &ctx->l_poses, &ctx->l_mt, &ctx->l_mtidx, &ctx->l_W,
                    &ctx->l_rew, &ctx->l_active, &ctx->l_nactive, &ctx->l_counters, &ctx->l_npose,
                    &ctx->l_nmeta, &ctx->b_counter, &ctx->l_push, &ctx->l_status, &ctx->l_stepping, &ctx->l_rec};
  for (DevBuf* b : bufs) b->release();
  ctx->b_pipe.release();
  for (cudaStream_t& s : ctx->pipe_stream)
    if (s) cudaStreamDestroy(s);
  if (ctx->pipe_ev) cudaEventDestroy(ctx->pipe_ev);
  dtree_release(ctx);
  for (int k = 0; k < kChunks; ++k) {
    ctx->chunk_in[k].release();
    ctx->chunk_buf[k].release();
    if (ctx->chunk_stream[k]) cudaStreamDestroy(ctx->chunk_stream[k]);
    if (ctx->chunk_ev[k]) cudaEventDestroy(ctx->chunk_ev[k]);
  }
  if (ctx->h_nactive) cudaFreeHost(ctx->h_nactive);
  if (ctx->h_epochs) cudaFreeHost(ctx->h_epochs);
  ctx->l_go.release();
  for (DevBuf* b : {&ctx->l_around, &ctx->l_astate, &ctx->l_aW, &ctx->l_actr, &ctx->l_adl, &ctx->l_actl, &ctx->trace_buf,
                    &ctx->l_fin, &ctx->l_rsi, &ctx->l_ract, &ctx->l_gring, &ctx->l_aP, &ctx->l_spec})
    b->release();
  if (ctx->h_go) cudaFreeHost(ctx->h_go);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

const char* ppg_last_error(ppg_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int ppg_set_params(ppg_ctx* ctx, const ppg_params* params) {
  if (!ctx || !params) return PPG_EINVAL;
  const int rc = check_params(ctx, *params);
  if (rc != PPG_SUCCESS) return rc;
  ctx->params = *params;
  if (ctx->group && ppg::group_member(ctx->group, 0) == ctx)  // the other shards of a multi-device context
    for (int k = 1; k < ppg::group_size(ctx->group); ++k) ppg::group_member(ctx->group, k)->params = *params;
  return PPG_SUCCESS;
}

int ppg_set_scene(ppg_ctx* ctx, const ppg_shapes* shapes) {
  if (!ctx || !shapes || shapes->n_tables != 1) return PPG_EINVAL;
  CK(cudaSetDevice(ctx->device));
  const int n = shapes->n_objects;
  if (ctx->has_scene && !ctx->group && static_cast<int>(ctx->h_kind.size()) == n && n > 0 &&
      ctx->side == shapes->side_length && ctx->margin == shapes->boundary_margin &&
      std::equal(ctx->h_kind.begin(), ctx->h_kind.end(), shapes->kind) &&
      std::memcmp(ctx->h_radius.data(), shapes->radius, n * sizeof(double)) == 0 &&
      ctx->h_target[0] == shapes->target_index[0] &&
      (shapes->n_vertices ? std::equal(ctx->h_nv.begin(), ctx->h_nv.end(), shapes->n_vertices)
                          : std::all_of(ctx->h_nv.begin(), ctx->h_nv.end(), [](int v) { return v == 0; })) &&
      (shapes->vertices ? std::memcmp(ctx->h_verts.data(), shapes->vertices, ctx->h_verts.size() * sizeof(double)) == 0
                        : std::all_of(ctx->h_verts.begin(), ctx->h_verts.end(), [](double v) { return v == 0.0; })))
    return PPG_SUCCESS;  // the installed scene already (run_pmbs installs the state's scene on every call)
  ctx->h_kind.assign(shapes->kind, shapes->kind + n);
  ctx->h_radius.assign(shapes->radius, shapes->radius + n);
  ctx->h_nv.assign(n, 0);
  if (shapes->n_vertices) ctx->h_nv.assign(shapes->n_vertices, shapes->n_vertices + n);
  ctx->h_verts.assign(static_cast<size_t>(n) * kMaxV * 2, 0.0);
  if (shapes->vertices) ctx->h_verts.assign(shapes->vertices, shapes->vertices + static_cast<size_t>(n) * kMaxV * 2);
  ctx->h_target.assign(shapes->target_index, shapes->target_index + 1);
  ctx->side = shapes->side_length;
  ctx->margin = shapes->boundary_margin;
  ctx->scene_all_discs = host_all_discs(shapes);
  const int rc = upload_shapes(ctx, shapes, false, ctx->scene_in, ctx->scene_buf, ctx->scene, ctx->stream);
  if (rc != PPG_SUCCESS) return rc;
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->has_scene = true;
  if (ctx->group && ppg::group_member(ctx->group, 0) == ctx)  // the other shards of a multi-device context
    for (int k = 1; k < ppg::group_size(ctx->group); ++k) {
      ppg_ctx* c = ppg::group_member(ctx->group, k);
      ppg::Group* g = c->group;
      c->group = nullptr;  // install on the member alone
      const int rc2 = ppg_set_scene(c, shapes);
      c->group = g;
      if (rc2 != PPG_SUCCESS) {
        ctx->err = c->err;
        return rc2;
      }
    }
  return PPG_SUCCESS;
}

}  // extern "C"

// Launches resolve_disc_kernel<N> (N = the smallest instantiated size >= n)
// as a persistent grid sized for `work` environments.  The work counter
// (ctx->b_counter) is zeroed here unless the caller's graph zeroes it.
int launch_disc(ppg_ctx* ctx, const SimConst& C, const ResolveArgs& a, int n, int work, cudaStream_t st,
                bool zero_counter, int slot_counter, bool fixpoint) {
  CK(ctx->b_counter.ensure(64));
  int* counter = ctx->b_counter.as<int>() + 4 * slot_counter;  // one counter per concurrent launch
  if (zero_counter) CK(cudaMemsetAsync(counter, 0, 4, st));
  int slot = 0;
  while (kDiscSizes[slot] < n) ++slot;
  const int nmax = kDiscSizes[slot];
  const int want = (work + kDiscBlock - 1) / kDiscBlock;
  const int bps = ctx->disc_bps_override > 0 && ctx->disc_bps_override < ctx->disc_blocks_per_sm[slot]
                      ? ctx->disc_bps_override
                      : ctx->disc_blocks_per_sm[slot];
  const int cap = bps * ctx->num_sms;
  // a batch that fills at least half the resident lanes gets one full wave
  // (every SM the same number of blocks; the kernel spreads the envs evenly)
  const int grid = want * 2 >= cap ? cap : (want < 1 ? 1 : want);
  const size_t sm = disc_smem(nmax);
#define PPG_DISC_LAUNCH(N)                                                              \
  (fixpoint ? resolve_disc_kernel<N, true><<<grid, kDiscBlock, sm, st>>>(C, a, counter)  \
            : resolve_disc_kernel<N, false><<<grid, kDiscBlock, sm, st>>>(C, a, counter))
  switch (nmax) {
    case 4: PPG_DISC_LAUNCH(4); break;
    case 6: PPG_DISC_LAUNCH(6); break;
    case 8: PPG_DISC_LAUNCH(8); break;
    case 10: PPG_DISC_LAUNCH(10); break;
    case 11: PPG_DISC_LAUNCH(11); break;
    case 12: PPG_DISC_LAUNCH(12); break;
    case 14: PPG_DISC_LAUNCH(14); break;
    case 16: PPG_DISC_LAUNCH(16); break;
    case 18: PPG_DISC_LAUNCH(18); break;
    default: PPG_DISC_LAUNCH(20); break;
  }
#undef PPG_DISC_LAUNCH
  CK(cudaGetLastError());
  return PPG_SUCCESS;
}

bool use_disc(const ppg_ctx* ctx, bool all_discs, int n) {
  return all_discs && n <= kDiscMaxN && ctx->disc_kernels && !ctx->force_generic;
}

// Latency mode (one warp per env, warp_env.cu) vs the lane-per-env kernels.
// For PMBS work (expansion, lockstep rounds: sample + pick + resolve + graspable per
// env-step) latency mode always wins — its sampler and graspable run across
// the lanes, and a round costs its slowest env-step (measured: case_18 at
// N_e = 16K, 1.02 s -> 0.44 s).  For plain batch_resolve throughput the
// lane-per-env disc kernel (discs, n <= kDiscMaxN) wins above 2,048 envs (measured
// with 10 and 16 discs); scenes without it (discs with n > 16, polygons) stay in latency mode.
// PPG_WARP_MAX, if set, caps latency mode everywhere.
bool use_warp(const ppg_ctx* ctx, bool all_discs, int n, int envs, bool pmbs) {
  if (ctx->force_generic) return false;
  const bool shape_ok = all_discs ? n <= kWarpMaxN : (ctx->warp_poly && n <= kPolyMaxN);
  if (!shape_ok) return false;
  if (ctx->warp_max_explicit) return envs <= ctx->warp_max_envs;
  if (!pmbs && all_discs && n <= kDiscMaxN && ctx->disc_kernels) return envs <= ctx->warp_max_envs;
  return true;
}

RoundMode round_mode(const ppg_ctx* ctx, int n, int envs) {
  if (use_warp(ctx, ctx->scene_all_discs, n, envs, true)) {
    const bool hybrid_ok = ctx->scene_all_discs && n <= kDiscMaxN && ctx->disc_kernels && !ctx->warp_max_explicit;
    return hybrid_ok && envs >= ctx->hybrid_min_envs ? RoundMode::kHybrid : RoundMode::kWarp;
  }
  if (use_disc(ctx, ctx->scene_all_discs, n)) return RoundMode::kLaneDisc;
  return RoundMode::kGeneric;
}

// One lockstep round (RolloutCursor::step for every active env) over the
// `work` envs the grids are sized for:
//  kWarp     one warp per env: sample + pick + resolve + graspable;
//  kHybrid   large disc batches: sample + pick one warp per env ->
//            resolve_disc lane kernel (in place) -> graspable one warp per env;
//  kLaneDisc the same three phases one lane per env;
//  kAdaptive kWarp and kHybrid kernels both launched, the harvest's
//            round_mode flag (n_active >= hybrid_min) selects one per round;
//  kGeneric  the straight one-lane transcription.
int lock_round_on(ppg_ctx* ctx, const SimConst& C, const LockArgs& a, const ResolveArgs& ra, int work,
                  RoundMode mode, cudaStream_t st) {
  const int n = ctx->scene.n;
  const int g = (work + kBlock - 1) / kBlock;
  const int gw = (work + kWarpsPerBlock - 1) / kWarpsPerBlock;
  switch (mode) {
    case RoundMode::kWarp:
      PPG_WARP_LAUNCH(lock_step_warp_kernel, !ctx->scene_all_discs, n, work, st, C, a);
      break;
    case RoundMode::kAdaptive:  // both; the harvest's round_mode flag picks (device tree)
      PPG_WARP_LAUNCH(lock_step_warp_kernel, false, n, work, st, C, a);
      CK(cudaGetLastError());
      [[fallthrough]];
    case RoundMode::kHybrid: {
      lock_sample_warp_kernel<<<gw, kWarpsPerBlock * 32, 0, st>>>(C, a);
      CK(cudaGetLastError());
      const int rc = launch_disc(ctx, C, ra, n, work, st);
      if (rc != PPG_SUCCESS) return rc;
      lock_post_warp_kernel<<<gw, kWarpsPerBlock * 32, 0, st>>>(C, a);
      break;
    }
    case RoundMode::kLaneDisc: {
      lock_sample_kernel<<<g, kBlock, smem_for(n), st>>>(C, a);
      CK(cudaGetLastError());
      const int rc = launch_disc(ctx, C, ra, n, work, st);
      if (rc != PPG_SUCCESS) return rc;
      lock_post_kernel<<<g, kBlock, smem_for(n), st>>>(C, a);
      break;
    }
    default:
      lock_step_kernel<<<g, kBlock, smem_for(n), st>>>(C, a);
  }
  CK(cudaGetLastError());
  return PPG_SUCCESS;
}

bool async_enabled(const ppg_ctx* ctx) {
  if (ctx->async_mode < 0) {
    const char* v = std::getenv("PPG_ASYNC");
    const_cast<ppg_ctx*>(ctx)->async_mode = (v && v[0] == '0') ? 0 : 1;
  }
  return ctx->async_mode == 1 && !ctx->force_generic;
}

template <int NW, bool kPoly>
static int launch_async_t(ppg_ctx* ctx, const SimConst& C, const LockArgs& a, int work, cudaStream_t st, bool cont) {
  static int bps[4] = {-1, -1, -1, -1};
  // speculative re-purposing compiled in only where it is used (a_spec set:
  // small batches); the plain instantiation keeps its registers
  const bool spec = a.a_spec != nullptr;
  const void* fn = spec ? reinterpret_cast<const void*>(&lock_async_kernel<NW, kPoly, true>)
                        : reinterpret_cast<const void*>(&lock_async_kernel<NW, kPoly, false>);
  int& b = bps[(kPoly ? 1 : 0) + (spec ? 2 : 0)];
  if (b < 0) {
    int v = 0;
    if (spec) CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, lock_async_kernel<NW, kPoly, true>, kWarpsPerBlock * 32, 0));
    else CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, lock_async_kernel<NW, kPoly, false>, kWarpsPerBlock * 32, 0));
    b = v > 0 ? v : 1;
  }
  const int want = (work + 1 + kWarpsPerBlock - 1) / kWarpsPerBlock;  // + the harvester warp
  const int grid = want < b * ctx->num_sms ? want : b * ctx->num_sms;
  if (!cont) {
    lock_async_init_kernel<<<(work + 255) / 256 + 1, 256, 0, st>>>(C, a);
    CK(cudaGetLastError());
  }
  // every warp must be resident (workers and the harvester wait on each other)
  SimConst c_arg = C;
  LockArgs a_arg = a;
  void* args[] = {&c_arg, &a_arg};
  CK(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kWarpsPerBlock * 32), args, 0, st));
  return PPG_SUCCESS;
}

bool speculate_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("PPG_SPECULATE");
    return !(v && v[0] == '0');
  }();
  return on;
}

bool wave_enabled(const ppg_ctx* ctx) {
  if (ctx->wave_mode < 0) {
    ppg_ctx* c = const_cast<ppg_ctx*>(ctx);
    const char* v = std::getenv("PPG_WAVE");
    c->wave_mode = (v && v[0] == '0') ? 0 : 1;
    const char* b = std::getenv("PPG_WAVE_BUDGET");
    if (b && std::atoi(b) > 0) c->wave_budget = std::atoi(b);
    const char* w = std::getenv("PPG_WAVE_SWITCH");
    if (w) c->wave_switch = std::atoi(w);
  }
  return ctx->wave_mode == 1 && async_enabled(ctx);
}

// One wave (see warp_env.cu): harvest of the complete rounds + lists, sample,
// budgeted lane physics (in place, resumable), post.  `work` sizes the grids.
int launch_wave(ppg_ctx* ctx, const SimConst& C, const LockArgs& a, const ResolveArgs& ra_in, int work,
                cudaStream_t st) {
  const int gw = (work + kWarpsPerBlock - 1) / kWarpsPerBlock;
  wave_harvest_kernel<<<1, 1024, 0, st>>>(C, a);
  CK(cudaGetLastError());
  wave_sample_kernel<<<gw, kWarpsPerBlock * 32, 0, st>>>(C, a);
  CK(cudaGetLastError());
  ResolveArgs ra = ra_in;
  ra.resume_si = a.resume_si;
  ra.resume_active = a.resume_active;
  ra.fin_list = a.fin_list;
  ra.fin_count = a.fin_count;
  ra.budget = ctx->wave_budget;
  ra.budget_dev = a.a_ctl + 8;  // set by the harvest: the budget, or unbounded in the hand-over wave
  const int rc = launch_disc(ctx, C, ra, ctx->scene.n, work, st, true, 0, true);
  if (rc != PPG_SUCCESS) return rc;
  wave_post_kernel<<<gw, kWarpsPerBlock * 32, 0, st>>>(C, a);
  CK(cudaGetLastError());
  return PPG_SUCCESS;
}

// cont: continue from a wave-round state (no re-initialisation)
int launch_async(ppg_ctx* ctx, const SimConst& C, const LockArgs& a, int work, cudaStream_t st, bool cont) {
  const int n = ctx->scene.n, w = warp_words(n);
  if (!ctx->scene_all_discs) {
    if (w == 1) return launch_async_t<1, true>(ctx, C, a, work, st, cont);
    if (w == 2) return launch_async_t<2, true>(ctx, C, a, work, st, cont);
    return launch_async_t<4, true>(ctx, C, a, work, st, cont);
  }
  if (w == 1) return launch_async_t<1, false>(ctx, C, a, work, st, cont);
  if (w == 2) return launch_async_t<2, false>(ctx, C, a, work, st, cont);
  if (w == 4) return launch_async_t<4, false>(ctx, C, a, work, st, cont);
  return launch_async_t<8, false>(ctx, C, a, work, st, cont);
}

// Polygon batches (one warp per env): past one resident wave the grid is
// persistent, warps taking envs from a counter (per-env cost varies by an
// order of magnitude; fixed 4-warp blocks idled on their slowest env).
template <int NW>
static int launch_resolve_poly_t(ppg_ctx* ctx, const SimConst& C, ResolveArgs a, int E, cudaStream_t st, int slot) {
  static int bps = -1;  // resident blocks per SM (a property of the kernel on this device)
  if (bps < 0) {
    int b = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, resolve_warp_kernel<NW, true>, kWarpsPerBlock * 32, 0));
    bps = b > 0 ? b : 1;
  }
  const int want = (E + kWarpsPerBlock - 1) / kWarpsPerBlock;
  const int cap = bps * ctx->num_sms;
  int grid = want;
  if (want > cap) {
    CK(ctx->b_counter.ensure(64));
    a.work_counter = ctx->b_counter.as<int>() + 4 * slot;
    CK(cudaMemsetAsync(a.work_counter, 0, 4, st));
    grid = cap;
    // more envs than resident warps: fetch the likely-heavy envs first
    // (poly_order_key_kernel; PPG_POLY_ORDER=0 keeps index order)
    static const bool order = [] {
      const char* v = std::getenv("PPG_POLY_ORDER");
      return !(v && v[0] == '0');
    }();
    if (order && !a.idx && !a.E_dev) {
      size_t scratch = 0;
      CK(cub::DeviceRadixSort::SortPairsDescending(nullptr, scratch, static_cast<const unsigned*>(nullptr),
                                                   static_cast<unsigned*>(nullptr), static_cast<const int*>(nullptr),
                                                   static_cast<int*>(nullptr), E, 0, 24, st));
      const size_t En = (static_cast<size_t>(E) + 63) / 64 * 64;
      CK(ctx->ord_buf[slot].ensure(4 * En * 4 + scratch));
      unsigned* k_in = ctx->ord_buf[slot].as<unsigned>();
      unsigned* k_out = k_in + En;
      int* v_in = reinterpret_cast<int*>(k_out + En);
      int* v_out = v_in + En;
      poly_order_key_kernel<<<(E + 255) / 256, 256, 0, st>>>(a, k_in, v_in);
      CK(cudaGetLastError());
      CK(cub::DeviceRadixSort::SortPairsDescending(v_out + En, scratch, k_in, k_out, v_in, v_out, E, 0, 24, st));
      a.idx = v_out;
    }
  }
  resolve_warp_kernel<NW, true><<<grid, kWarpsPerBlock * 32, 0, st>>>(C, a);
  CK(cudaGetLastError());
  return PPG_SUCCESS;
}

static int launch_resolve_poly(ppg_ctx* ctx, const SimConst& C, const ResolveArgs& a, int n, int E, cudaStream_t st,
                               int slot) {
  const int w = warp_words(n);
  if (w == 1) return launch_resolve_poly_t<1>(ctx, C, a, E, st, slot);
  if (w == 2) return launch_resolve_poly_t<2>(ctx, C, a, E, st, slot);
  return launch_resolve_poly_t<4>(ctx, C, a, E, st, slot);
}

// Kernel #1 dispatch: all-disc batches (shapes without vertex tables) run the
// register-resident persistent kernel (resolve_disc.cu) sized to the object
// count; polygons, n > 16 and the counting variant run the generic kernel.
static int launch_resolve(ppg_ctx* ctx, const ShapesDev& S, bool all_discs, double side, double margin,
                          const double* d_in, const double* d_push, int E, double* d_out, int32_t* d_status,
                          double* d_resid, long long* d_counts, cudaStream_t st, int slot = 0) {
  const SimConst C = make_const(ctx->params, S.n, side, margin);
  ResolveArgs a{S, d_in, d_push, d_out, d_status, d_resid, d_counts, E};
  if (!d_counts && use_warp(ctx, all_discs, S.n, E, false)) {
    if (!all_discs) return launch_resolve_poly(ctx, C, a, S.n, E, st, slot);
    PPG_WARP_LAUNCH(resolve_warp_kernel, false, S.n, E, st, C, a);
    CK(cudaGetLastError());
    return PPG_SUCCESS;
  }
  if (!d_counts && use_disc(ctx, all_discs, S.n)) return launch_disc(ctx, C, a, S.n, E, st, true, slot, false);
  const int grid = (E + kBlock - 1) / kBlock;
  if (d_counts) resolve_kernel<true><<<grid, kBlock, smem_for(S.n), st>>>(C, a);
  else resolve_kernel<false><<<grid, kBlock, smem_for(S.n), st>>>(C, a);
  CK(cudaGetLastError());
  return PPG_SUCCESS;
}



extern "C" {

// Large host-buffer batches are split into kChunks slices processed on
// separate streams, so the host<->device copies of one slice overlap the
// physics of the others (the element-wise results are independent of the
// split).  Below this size one launch on the context stream.
constexpr int kPipelineMinEnvs = 32768;

static int batch_resolve_chunk(ppg_ctx* ctx, const ppg_shapes* shapes, const double* poses_in,
                               const double* pushes, int e0, int e1, double* poses_out, int32_t* status,
                               double* residual, cudaStream_t st, int slot, cudaEvent_t after = nullptr,
                               cudaEvent_t h2d_done = nullptr) {
  const int Ek = e1 - e0;
  // host->device copies in slice order (slice k's physics overlaps slice
  // k+1's copies instead of every slice waiting for interleaved copies)
  if (after) CK(cudaStreamWaitEvent(st, after, 0));
  ShapesDev S;
  double side, margin;
  bool discs;
  if (shapes) {
    ppg_shapes sub = *shapes;
    if (shapes->n_tables != 1) {  // this slice's tables
      const size_t n = static_cast<size_t>(shapes->n_objects);
      sub.n_tables = Ek;
      sub.kind = shapes->kind + e0 * n;
      sub.radius = shapes->radius + e0 * n;
      sub.n_vertices = shapes->n_vertices ? shapes->n_vertices + e0 * n : nullptr;
      sub.vertices = shapes->vertices ? shapes->vertices + e0 * n * kMaxV * 2 : nullptr;
      sub.target_index = shapes->target_index + e0;
    }
    const int rc = upload_shapes(ctx, &sub, false, ctx->chunk_in[slot], ctx->chunk_buf[slot], S, st);
    if (rc != PPG_SUCCESS) return rc;
    side = shapes->side_length;
    margin = shapes->boundary_margin;
    discs = host_all_discs(&sub);
  } else {
    S = ctx->scene;
    side = ctx->side;
    margin = ctx->margin;
    discs = ctx->scene_all_discs;
  }
  const size_t row = static_cast<size_t>(S.n) * 3;
  double* d_in = ctx->b_in.as<double>() + e0 * row;
  double* d_out = ctx->b_out.as<double>() + e0 * row;
  double* d_push = ctx->b_push.as<double>() + e0 * 4ull;
  int32_t* d_st = ctx->b_status.as<int32_t>() + e0;
  double* d_res = ctx->b_resid.as<double>() + e0;
  CK(cudaMemcpyAsync(d_in, poses_in + e0 * row, Ek * row * 8, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_push, pushes + e0 * 4ull, Ek * 32ull, cudaMemcpyHostToDevice, st));
  if (h2d_done) CK(cudaEventRecord(h2d_done, st));
  const int rc = launch_resolve(ctx, S, discs, side, margin, d_in, d_push, Ek, d_out, d_st, d_res, nullptr, st, slot);
  if (rc != PPG_SUCCESS) return rc;
  CK(cudaMemcpyAsync(poses_out + e0 * row, d_out, Ek * row * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(status + e0, d_st, Ek * 4ull, cudaMemcpyDeviceToHost, st));
  if (residual) CK(cudaMemcpyAsync(residual + e0, d_res, Ek * 8ull, cudaMemcpyDeviceToHost, st));
  return PPG_SUCCESS;
}

// Device address of a mapped pinned host buffer, or null (pageable memory).
static void* mapped_host(const void* p) {
  if (!p) return nullptr;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return at.type == cudaMemoryTypeHost ? at.devicePointer : nullptr;
}

using WriteValue32Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using WaitValue32Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

// Probes the streamed path once per context: PPG_STREAMED=0 disables it;
// it needs the driver's stream memory operations.
static bool streamed_available(ppg_ctx* ctx) {
  if (ctx->streamed >= 0) return ctx->streamed == 1;
  ctx->streamed = 0;
  const char* v = std::getenv("PPG_STREAMED");
  if (v && v[0] == '0') return false;
  cudaDriverEntryPointQueryResult q1{}, q2{};
  if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &ctx->fn_write32, cudaEnableDefault, &q1) != cudaSuccess ||
      cudaGetDriverEntryPoint("cuStreamWaitValue32", &ctx->fn_wait32, cudaEnableDefault, &q2) != cudaSuccess ||
      q1 != cudaDriverEntryPointSuccess || q2 != cudaDriverEntryPointSuccess || !ctx->fn_write32 || !ctx->fn_wait32) {
    cudaGetLastError();
    return false;
  }
  for (cudaStream_t& st : ctx->pipe_stream)
    if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return false;
  if (cudaEventCreateWithFlags(&ctx->pipe_ev, cudaEventDisableTiming) != cudaSuccess) return false;
  if (ctx->b_pipe.ensure(2 * kMaxSlices * sizeof(unsigned)) != cudaSuccess ||
      cudaMemset(ctx->b_pipe.p, 0, 2 * kMaxSlices * sizeof(unsigned)) != cudaSuccess)
    return false;
  if (!ctx->h_epochs && cudaMallocHost(&ctx->h_epochs, kMaxSlices * sizeof(unsigned)) != cudaSuccess) return false;
  ctx->streamed = 1;
  return true;
}

// Waits for the streamed physics launch with a bound: every slice copy and
// ready-flag write is enqueued before the launch, so lanes waiting on a flag
// always get it — unless that invariant is ever broken.  Then, instead of a
// hung GPU, the flags are released from a side stream (the lanes finish on
// whatever the buffers hold) and the call reports an error.
static int wait_streamed(ppg_ctx* ctx, cudaStream_t ph, unsigned* ready, unsigned epoch) {
  static const double limit = [] {
    const char* v = std::getenv("PPG_STREAM_TIMEOUT_S");
    return v ? std::atof(v) : 120.0;
  }();
  const auto t0 = std::chrono::steady_clock::now();
  for (int spins = 0;; ++spins) {
    const cudaError_t e = cudaStreamQuery(ph);
    if (e == cudaSuccess) return PPG_SUCCESS;
    if (e != cudaErrorNotReady) {
      ctx->err = std::string("streamed batch_resolve: ") + cudaGetErrorString(e);
      return PPG_ECUDA;
    }
    // poll without sleeping for the first 20 ms (a sleep costs ~50-80 us of
    // timer slack at the end of a ~1.7 ms call), then back off
    const double waited = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (waited > 0.02) std::this_thread::sleep_for(std::chrono::microseconds(20));
    else if (spins > 64) std::this_thread::yield();
    if (waited > limit) {
      cudaStream_t rescue = nullptr;
      std::vector<unsigned> fl(kMaxSlices, epoch);
      if (cudaStreamCreateWithFlags(&rescue, cudaStreamNonBlocking) == cudaSuccess) {
        cudaMemcpyAsync(ready, fl.data(), kMaxSlices * sizeof(unsigned), cudaMemcpyHostToDevice, rescue);
        cudaStreamSynchronize(ph);
        cudaStreamDestroy(rescue);
      }
      ctx->err = "streamed batch_resolve: slice ready flags never arrived (PPG_STREAM_TIMEOUT_S); released";
      return PPG_ECUDA;
    }
  }
}

// Streamed host-buffer batch_resolve for disc batches: ONE persistent physics
// launch (resolve_disc_kernel) overlaps every host<->device copy.
//   copy-in stream: per slice, poses + pushes + radii (the host [E][n] radius
//     layout is read as is: no shape transpose, no kind/target upload), then
//     a stream write of `epoch` into the slice's ready flag;
//   physics stream: launched once slice 0 is resident; lanes take envs in
//     slice order and wait on the flag of an env's slice before loading it;
//     every finished env bumps its slice's done counter;
//   output: when poses_out / status / residual are pinned host buffers the
//     kernel writes them directly (each finished env's poses in one
//     warp-coalesced write), so the copy-back overlaps the physics env by env
//     (PPG_ZC_OUT=0 disables); otherwise a copy-out stream waits per slice
//     until the done counter reaches the slice's size and copies it back.
// Results are element-wise, identical to the one-launch path
// (tests/test_gpu_parity.py).
static int batch_resolve_streamed(ppg_ctx* ctx, const ppg_shapes* sh, const double* poses_in, const double* pushes,
                                  int E, double* poses_out, int32_t* status, double* residual) {
  const int n = sh->n_objects;
  const size_t row = static_cast<size_t>(n) * 3;
  static const int per_slice = [] {
    const char* v = std::getenv("PPG_SLICE_ENVS");  // experiments; default 16K envs per slice (measured best of 4K-32K)
    return v && std::atoi(v) >= 256 ? std::atoi(v) : 16384;
  }();
  // PPG_SLICE_SCHED=0: uniform slices of PPG_SLICE_ENVS, each copied on its
  // own.  Default (tapered): the kernel sees kMaxSlices small slices, copied
  // in groups that shrink toward the end of the batch (big early groups,
  // single slices last), so the envs that land last are few and the batch's
  // tail (the heaviest env of the last-landing group) starts early.
  static const bool tapered = [] {
    const char* v = std::getenv("PPG_SLICE_SCHED");
    return !(v && v[0] == '0');
  }();
  const int want = tapered ? (E + 2047) / 2048 : (E + per_slice - 1) / per_slice;
  const int slices = want < 2 ? 2 : (want > kMaxSlices ? kMaxSlices : want);
  // multiples of 16 envs: no cache line of any input array spans two slices
  const int slice_envs = ((E + slices - 1) / slices + 15) / 16 * 16;
  const int ns = (E + slice_envs - 1) / slice_envs;
  int group_end[kMaxSlices];  // copy groups: slices [group_end[g-1], group_end[g])
  int ng = 0;
  if (tapered) {  // ns = 32: 8 8 6 4 3 2 1 slices
    const int g0 = ns / 4 > 1 ? ns / 4 : 1;
    for (int k = 0, g = g0, i = 0; k < ns; ++i) {
      k = k + g < ns ? k + g : ns;
      group_end[ng++] = k;
      if (i > 0) g = g * 3 / 4 > 1 ? g * 3 / 4 : 1;
    }
  } else {
    for (int k = 1; k <= ns; ++k) group_end[ng++] = k;
  }
  CK(ctx->shape_in.ensure(static_cast<size_t>(E) * n * sizeof(double)));
  double* rad = ctx->shape_in.as<double>();
  unsigned* ready = ctx->b_pipe.as<unsigned>();
  unsigned* done = ready + kMaxSlices;
  const unsigned epoch = ++ctx->pipe_epoch == 0 ? ++ctx->pipe_epoch : ctx->pipe_epoch;
  auto write32 = reinterpret_cast<WriteValue32Fn>(ctx->fn_write32);
  auto wait32 = reinterpret_cast<WaitValue32Fn>(ctx->fn_wait32);
  cudaStream_t in = ctx->pipe_stream[0], ph = ctx->pipe_stream[1], out = ctx->pipe_stream[2];
  int* counter = ctx->b_counter.as<int>();
  CK(cudaStreamSynchronize(ctx->stream));  // earlier work on the context stream
  // PPG_STREAM_TRACE=1: per-stage event times to stderr (experiments)
  static const bool trace = std::getenv("PPG_STREAM_TRACE") != nullptr;
  cudaEvent_t tev[2 * kMaxSlices + 4] = {};
  int ntev = 0;
  auto mark = [&](cudaStream_t s) {
    if (!trace) return;
    cudaEventCreate(&tev[ntev]);
    cudaEventRecord(tev[ntev++], s);
  };
  mark(in);
  CK(cudaMemsetAsync(done, 0, kMaxSlices * sizeof(unsigned), in));
  CK(cudaMemsetAsync(counter, 0, 4, in));
  double* d_in = ctx->b_in.as<double>();
  double* d_out = ctx->b_out.as<double>();
  double* d_push = ctx->b_push.as<double>();
  int32_t* d_st = ctx->b_status.as<int32_t>();
  double* d_res = ctx->b_resid.as<double>();
  // ready flags: one small pinned-host copy per group (default) or one
  // cuStreamWriteValue32 per slice (PPG_SLICE_FLAGS=m); measured 1.5 % apart
  static const bool flag_copy = [] {
    const char* v = std::getenv("PPG_SLICE_FLAGS");
    return !(v && v[0] == 'm');
  }();
  if (flag_copy)
    for (int k = 0; k < kMaxSlices; ++k) ctx->h_epochs[k] = epoch;  // the previous call's copies are complete
  for (int g = 0; g < ng; ++g) {
    const int k0 = g ? group_end[g - 1] : 0, k1 = group_end[g];
    const size_t e0 = static_cast<size_t>(k0) * slice_envs;
    const size_t ek = (k1 == ns ? E : static_cast<size_t>(k1) * slice_envs) - e0;
    CK(cudaMemcpyAsync(d_in + e0 * row, poses_in + e0 * row, ek * row * 8, cudaMemcpyHostToDevice, in));
    CK(cudaMemcpyAsync(d_push + e0 * 4, pushes + e0 * 4, ek * 32, cudaMemcpyHostToDevice, in));
    CK(cudaMemcpyAsync(rad + e0 * n, sh->radius + e0 * n, ek * n * 8, cudaMemcpyHostToDevice, in));
    if (flag_copy) {  // the group's ready flags in one copy, ordered after its data on the stream
      CK(cudaMemcpyAsync(ready + k0, ctx->h_epochs, (k1 - k0) * sizeof(unsigned), cudaMemcpyHostToDevice, in));
    } else {
      for (int k = k0; k < k1; ++k)
        if (write32(reinterpret_cast<CUstream>(in), reinterpret_cast<CUdeviceptr>(ready + k), epoch,
                    CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS) {
          ctx->err = "cuStreamWriteValue32 failed";
          return PPG_ECUDA;
        }
    }
    if (g == 0) CK(cudaEventRecord(ctx->pipe_ev, in));
    mark(in);
  }
  // physics: one launch over all E envs once slice 0 is resident
  CK(cudaStreamWaitEvent(ph, ctx->pipe_ev, 0));
  const SimConst C = make_const(ctx->params, n, sh->side_length, sh->boundary_margin);
  ShapesDev S;
  S.rad = rad;
  S.T = E;
  S.n = n;
  ResolveArgs a{S, d_in, d_push, d_out, d_st, d_res, nullptr, E};
  a.ready = ready;
  a.done = done;
  a.epoch = epoch;
  a.slice_envs = slice_envs;
  a.rad_env_major = true;
  static const bool zc_ok = [] {
    const char* v = std::getenv("PPG_ZC_OUT");
    return !(v && v[0] == '0');
  }();
  void* m_out = zc_ok ? mapped_host(poses_out) : nullptr;
  void* m_st = zc_ok ? mapped_host(status) : nullptr;
  void* m_res = zc_ok && residual ? mapped_host(residual) : nullptr;
  if (m_out && m_st && (m_res || !residual)) {
    a.poses_out = static_cast<double*>(m_out);
    a.status = static_cast<int32_t*>(m_st);
    a.residual = static_cast<double*>(m_res);
    a.zc_out = true;
    a.done = nullptr;
  }
  const int rc = launch_disc(ctx, C, a, n, E, ph, false, 0, false);
  if (rc != PPG_SUCCESS) return rc;
  mark(ph);
  if (a.zc_out) {
    if (const int wrc = wait_streamed(ctx, ph, ready, epoch); wrc != PPG_SUCCESS) return wrc;
    CK(cudaStreamSynchronize(in));
    if (trace) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, tev[0], tev[ntev - 1]);
      std::fprintf(stderr, "stream trace (zero-copy out): kernel done %.3f ms\n", ms);
      for (int i = 0; i < ntev; ++i) cudaEventDestroy(tev[i]);
    }
    return PPG_SUCCESS;
  }
  // copy-out, slice by slice as each completes
  CK(cudaStreamWaitEvent(out, ctx->pipe_ev, 0));  // after the done counters were zeroed
  for (int k = 0; k < ns; ++k) {
    const size_t e0 = static_cast<size_t>(k) * slice_envs;
    const size_t ek = (k + 1 == ns ? E : e0 + slice_envs) - e0;
    if (wait32(reinterpret_cast<CUstream>(out), reinterpret_cast<CUdeviceptr>(done + k), static_cast<cuuint32_t>(ek),
               CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS) {
      ctx->err = "cuStreamWaitValue32 failed";
      return PPG_ECUDA;
    }
    CK(cudaMemcpyAsync(poses_out + e0 * row, d_out + e0 * row, ek * row * 8, cudaMemcpyDeviceToHost, out));
    CK(cudaMemcpyAsync(status + e0, d_st + e0, ek * 4, cudaMemcpyDeviceToHost, out));
    if (residual) CK(cudaMemcpyAsync(residual + e0, d_res + e0, ek * 8, cudaMemcpyDeviceToHost, out));
    mark(out);
  }
  if (const int wrc = wait_streamed(ctx, ph, ready, epoch); wrc != PPG_SUCCESS) return wrc;
  CK(cudaStreamSynchronize(out));
  if (trace) {
    std::fprintf(stderr, "stream trace (ms from start): in");
    for (int i = 1; i < ntev; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, tev[0], tev[i]);
      std::fprintf(stderr, i == ng + 1 ? " | kernel %.3f | out" : " %.3f", ms);
    }
    std::fprintf(stderr, "\n");
    for (int i = 0; i < ntev; ++i) cudaEventDestroy(tev[i]);
  }
  return PPG_SUCCESS;
}

int ppg_batch_resolve(ppg_ctx* ctx, const ppg_shapes* shapes, const double* poses_in, const double* pushes,
                      int E, double* poses_out, int32_t* status, double* residual) {
  if (!ctx || E < 0) return PPG_EINVAL;
  if (E == 0) return PPG_SUCCESS;
  CK(cudaSetDevice(ctx->device));
  if (shapes) {
    if (shapes->n_tables != 1 && shapes->n_tables != E) {
      ctx->err = "batch_resolve: states and shape tables must have equal length";
      return PPG_EINVAL;
    }
    if (shapes->n_objects < 1 || shapes->n_objects > kMaxObjects) {
      ctx->err = "n_objects must be in [1, 32] and n_tables >= 1";
      return PPG_EINVAL;
    }
  } else if (!ctx->has_scene) {
    ctx->err = "no scene installed";
    return PPG_EINVAL;
  }
  const int n = shapes ? shapes->n_objects : ctx->scene.n;
  const size_t pbytes = static_cast<size_t>(E) * n * 3 * sizeof(double);
  CK(ctx->b_in.ensure(pbytes));
  CK(ctx->b_out.ensure(pbytes));
  CK(ctx->b_push.ensure(static_cast<size_t>(E) * 4 * sizeof(double)));
  CK(ctx->b_status.ensure(static_cast<size_t>(E) * sizeof(int32_t)));
  CK(ctx->b_resid.ensure(static_cast<size_t>(E) * sizeof(double)));
  CK(ctx->b_counter.ensure(64));
  if (E >= kPipelineMinEnvs && shapes && shapes->n_tables == E && host_all_discs(shapes) && use_disc(ctx, true, n) &&
      !use_warp(ctx, true, n, E, false) && streamed_available(ctx))
    return batch_resolve_streamed(ctx, shapes, poses_in, pushes, E, poses_out, status, residual);
  const int chunks = E >= kPipelineMinEnvs ? kChunks : 1;
  if (chunks == 1) {
    int rc = batch_resolve_chunk(ctx, shapes, poses_in, pushes, 0, E, poses_out, status, residual, ctx->stream, 0);
    if (rc != PPG_SUCCESS) return rc;
    CK(cudaStreamSynchronize(ctx->stream));
    return PPG_SUCCESS;
  }
  for (int k = 0; k < chunks; ++k) {
    if (!ctx->chunk_stream[k]) CK(cudaStreamCreateWithFlags(&ctx->chunk_stream[k], cudaStreamNonBlocking));
    if (!ctx->chunk_ev[k]) CK(cudaEventCreateWithFlags(&ctx->chunk_ev[k], cudaEventDisableTiming));
  }
  CK(cudaStreamSynchronize(ctx->stream));  // earlier work on the context stream
  for (int k = 0; k < chunks; ++k) {
    const int e0 = static_cast<int>(static_cast<long long>(E) * k / chunks);
    const int e1 = static_cast<int>(static_cast<long long>(E) * (k + 1) / chunks);
    const int rc = batch_resolve_chunk(ctx, shapes, poses_in, pushes, e0, e1, poses_out, status, residual,
                                       ctx->chunk_stream[k], k, k ? ctx->chunk_ev[k - 1] : nullptr,
                                       ctx->chunk_ev[k]);
    if (rc != PPG_SUCCESS) return rc;
  }
  for (int k = 0; k < chunks; ++k) CK(cudaStreamSynchronize(ctx->chunk_stream[k]));
  return PPG_SUCCESS;
}

int ppg_batch_resolve_dev(ppg_ctx* ctx, const ppg_shapes* shapes_dev, const double* poses_in, const double* pushes,
                          int E, double* poses_out, int32_t* status, double* residual, void* stream) {
  if (!ctx || !shapes_dev || E < 0) return PPG_EINVAL;
  if (E == 0) return PPG_SUCCESS;
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool discs = !shapes_dev->n_vertices && !shapes_dev->vertices;  // documented contract
  const int n = shapes_dev->n_objects;
  if (discs && shapes_dev->n_tables == E && n >= 1 && n <= kMaxObjects && use_disc(ctx, true, n) &&
      !use_warp(ctx, true, n, E, false)) {
    // the lane-per-env disc kernel reads the caller's [E][n] radius table as
    // is (env-major strides): no shape-table transpose / vertex-table fill
    ShapesDev S;
    S.rad = const_cast<double*>(shapes_dev->radius);
    S.T = E;
    S.n = n;
    ResolveArgs a{S, poses_in, pushes, poses_out, status, residual, nullptr, E};
    a.rad_env_major = true;
    const SimConst C = make_const(ctx->params, n, shapes_dev->side_length, shapes_dev->boundary_margin);
    return launch_disc(ctx, C, a, n, E, st, true, 0, false);
  }
  ShapesDev S;
  const int rc = upload_shapes(ctx, shapes_dev, true, ctx->shape_in, ctx->shape_buf, S, st);
  if (rc != PPG_SUCCESS) return rc;
  return launch_resolve(ctx, S, discs, shapes_dev->side_length, shapes_dev->boundary_margin, poses_in, pushes, E,
                        poses_out, status, residual, nullptr, st);
}

int ppg_batch_resolve_count_dev(ppg_ctx* ctx, const ppg_shapes* shapes_dev, const double* poses_in,
                                const double* pushes, int E, int64_t* counts_dev, void* stream) {
  if (!ctx || !shapes_dev || E < 0) return PPG_EINVAL;
  if (E == 0) return PPG_SUCCESS;
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  ShapesDev S;
  int rc = upload_shapes(ctx, shapes_dev, true, ctx->shape_in, ctx->shape_buf, S, st);
  if (rc != PPG_SUCCESS) return rc;
  const size_t pbytes = static_cast<size_t>(E) * S.n * 3 * sizeof(double);
  CK(ctx->b_out.ensure(pbytes));
  CK(ctx->b_status.ensure(static_cast<size_t>(E) * 4));
  return launch_resolve(ctx, S, false, shapes_dev->side_length, shapes_dev->boundary_margin, poses_in, pushes, E,
                        ctx->b_out.as<double>(), ctx->b_status.as<int32_t>(), nullptr,
                        reinterpret_cast<long long*>(counts_dev), st);
}

// sample_pushes / graspable of small batches one warp per state
// (sample_grasp_warp_kernel); large batches one lane per state.
static bool sample_warp_ok(const ppg_ctx* ctx, bool all_discs, int n, int E) {
  const char* v = std::getenv("PPG_SAMPLE_WARP_MAX");
  const int emax = v ? std::atoi(v) : 8192;
  return E <= emax && n <= (all_discs ? kWarpMaxN : kPolyMaxN) && n * ctx->params.pushes_per_object <= 32 * 32;
}

static void launch_sample_grasp(const SimConst& C, const SampleArgs& a, bool all_discs, int E, cudaStream_t st) {
  const int grid = (E + kWarpsPerBlock - 1) / kWarpsPerBlock;
  if (all_discs) sample_grasp_warp_kernel<false><<<grid, kWarpsPerBlock * 32, 0, st>>>(C, a);
  else sample_grasp_warp_kernel<true><<<grid, kWarpsPerBlock * 32, 0, st>>>(C, a);
}

int ppg_sample_pushes(ppg_ctx* ctx, const ppg_shapes* shapes, const double* poses, int E, double* out,
                      int32_t* count) {
  if (!ctx || E < 0) return PPG_EINVAL;
  if (!shapes && !ctx->has_scene) {
    ctx->err = "no scene installed";
    return PPG_EINVAL;
  }
  if (E == 0) return PPG_SUCCESS;
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  ShapesDev S = ctx->scene;
  double side = ctx->side, margin = ctx->margin;
  if (shapes) {
    if (shapes->n_tables != 1 && shapes->n_tables != E) {
      ctx->err = "sample_pushes: shape tables must be 1 or E";
      return PPG_EINVAL;
    }
    const int rc = upload_shapes(ctx, shapes, false, ctx->shape_in, ctx->shape_buf, S, st);
    if (rc != PPG_SUCCESS) return rc;
    side = shapes->side_length;
    margin = shapes->boundary_margin;
  }
  const int n = S.n, na = ctx->params.pushes_per_object;
  const size_t pbytes = static_cast<size_t>(E) * n * 3 * 8, obytes = static_cast<size_t>(E) * n * na * 4 * 8;
  CK(ctx->b_in.ensure(pbytes));
  CK(ctx->b_out.ensure(obytes));
  CK(ctx->b_status.ensure(static_cast<size_t>(E) * 4));
  CK(cudaMemcpyAsync(ctx->b_in.p, poses, pbytes, cudaMemcpyHostToDevice, st));
  const SimConst C = make_const(ctx->params, n, side, margin);
  SampleArgs a{S, ctx->b_in.as<double>(), ctx->b_out.as<double>(), ctx->b_status.as<int32_t>(),
               nullptr, nullptr, nullptr, nullptr, nullptr, E};
  const bool discs = shapes ? host_all_discs(shapes) : ctx->scene_all_discs;
  if (sample_warp_ok(ctx, discs, n, E)) launch_sample_grasp(C, a, discs, E, st);
  else sample_kernel<<<(E + kBlock - 1) / kBlock, kBlock, smem_for(n), st>>>(C, a);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, ctx->b_out.p, obytes, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(count, ctx->b_status.p, static_cast<size_t>(E) * 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return PPG_SUCCESS;
}

// The search root's sample_pushes + graspable (SearchTree::create,
// mcts.cpp:28-39) in ONE launch and one synchronisation (run_pmbs setup).
int ppg_root_sample_grasp(ppg_ctx* ctx, const double* poses, double* untried, int32_t* count, uint8_t* graspable,
                          const double** untried_dev) {
  if (untried_dev) *untried_dev = nullptr;
  if (!ctx->has_scene) {
    ctx->err = "no scene installed";
    return PPG_EINVAL;
  }
  const int n = ctx->scene.n;
  if (!sample_warp_ok(ctx, ctx->scene_all_discs, n, 1)) {
    int rc = ppg_sample_pushes(ctx, nullptr, poses, 1, untried, count);
    if (rc == PPG_SUCCESS) rc = ppg_graspable(ctx, poses, 1, graspable, nullptr, nullptr, nullptr, nullptr);
    return rc;
  }
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  const int na = ctx->params.pushes_per_object;
  const size_t pbytes = static_cast<size_t>(n) * 3 * 8, obytes = static_cast<size_t>(n) * na * 4 * 8;
  CK(ctx->b_in.ensure(pbytes));
  CK(ctx->b_out.ensure(obytes));
  CK(ctx->b_status.ensure(64));
  CK(ctx->b_a.ensure(64));
  CK(ctx->b_b.ensure(64));
  CK(ctx->b_c.ensure(64));
  CK(ctx->b_d.ensure(64));
  CK(ctx->b_e.ensure(64));
  CK(cudaMemcpyAsync(ctx->b_in.p, poses, pbytes, cudaMemcpyHostToDevice, st));
  const SimConst C = make_const(ctx->params, n, ctx->side, ctx->margin);
  SampleArgs a{ctx->scene, ctx->b_in.as<double>(), ctx->b_out.as<double>(), ctx->b_status.as<int32_t>(),
               ctx->b_a.as<uint8_t>(), ctx->b_b.as<double>(), ctx->b_c.as<double>(), ctx->b_d.as<double>(),
               ctx->b_e.as<int32_t>(), 1};
  launch_sample_grasp(C, a, ctx->scene_all_discs, 1, st);
  CK(cudaGetLastError());
  if (untried_dev) {
    *untried_dev = ctx->b_out.as<double>();  // the caller copies it on the device
  } else {
    CK(cudaMemcpyAsync(untried, ctx->b_out.p, obytes, cudaMemcpyDeviceToHost, st));
  }
  CK(cudaMemcpyAsync(count, ctx->b_status.p, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(graspable, ctx->b_a.p, 1, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return PPG_SUCCESS;
}

int ppg_graspable(ppg_ctx* ctx, const double* poses, int E, uint8_t* graspable, double* margin, double* best_x,
                  double* best_y, int32_t* best_angle) {
  if (!ctx || E < 0) return PPG_EINVAL;
  if (!ctx->has_scene) {
    ctx->err = "no scene installed";
    return PPG_EINVAL;
  }
  if (E == 0) return PPG_SUCCESS;
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  const int n = ctx->scene.n;
  const size_t pbytes = static_cast<size_t>(E) * n * 3 * 8;
  CK(ctx->b_in.ensure(pbytes));
  CK(ctx->b_a.ensure(E));
  CK(ctx->b_b.ensure(static_cast<size_t>(E) * 8));
  CK(ctx->b_c.ensure(static_cast<size_t>(E) * 8));
  CK(ctx->b_d.ensure(static_cast<size_t>(E) * 8));
  CK(ctx->b_e.ensure(static_cast<size_t>(E) * 4));
  CK(cudaMemcpyAsync(ctx->b_in.p, poses, pbytes, cudaMemcpyHostToDevice, st));
  const SimConst C = make_const(ctx->params, n, ctx->side, ctx->margin);
  SampleArgs a{ctx->scene, ctx->b_in.as<double>(), nullptr, nullptr, ctx->b_a.as<uint8_t>(),
               ctx->b_b.as<double>(), ctx->b_c.as<double>(), ctx->b_d.as<double>(), ctx->b_e.as<int32_t>(), E};
  if (sample_warp_ok(ctx, ctx->scene_all_discs, n, E)) launch_sample_grasp(C, a, ctx->scene_all_discs, E, st);
  else grasp_kernel<<<(E + kBlock - 1) / kBlock, kBlock, smem_for(n), st>>>(C, a);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(graspable, ctx->b_a.p, E, cudaMemcpyDeviceToHost, st));
  if (margin) CK(cudaMemcpyAsync(margin, ctx->b_b.p, static_cast<size_t>(E) * 8, cudaMemcpyDeviceToHost, st));
  if (best_x) CK(cudaMemcpyAsync(best_x, ctx->b_c.p, static_cast<size_t>(E) * 8, cudaMemcpyDeviceToHost, st));
  if (best_y) CK(cudaMemcpyAsync(best_y, ctx->b_d.p, static_cast<size_t>(E) * 8, cudaMemcpyDeviceToHost, st));
  if (best_angle) CK(cudaMemcpyAsync(best_angle, ctx->b_e.p, static_cast<size_t>(E) * 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return PPG_SUCCESS;
}

int ppg_expand(ppg_ctx* ctx, const double* parent_poses, const double* actions, int P, double* child_poses,
               int32_t* status, uint8_t* graspable, int32_t* n_untried, double* untried) {
  if (!ctx || P < 0) return PPG_EINVAL;
  if (!ctx->has_scene) {
    ctx->err = "no scene installed";
    return PPG_EINVAL;
  }
  if (P == 0) return PPG_SUCCESS;
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  const int n = ctx->scene.n, na = ctx->params.pushes_per_object;
  const size_t pbytes = static_cast<size_t>(P) * n * 3 * 8, ubytes = static_cast<size_t>(P) * n * na * 4 * 8;
  CK(ctx->b_in.ensure(pbytes));
  CK(ctx->b_out.ensure(pbytes));
  CK(ctx->b_push.ensure(static_cast<size_t>(P) * 32));
  CK(ctx->b_status.ensure(static_cast<size_t>(P) * 4));
  CK(ctx->b_a.ensure(P));
  CK(ctx->b_e.ensure(static_cast<size_t>(P) * 4));
  CK(ctx->b_b.ensure(ubytes));
  CK(cudaMemcpyAsync(ctx->b_in.p, parent_poses, pbytes, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(ctx->b_push.p, actions, static_cast<size_t>(P) * 32, cudaMemcpyHostToDevice, st));
  const SimConst C = make_const(ctx->params, n, ctx->side, ctx->margin);
  ExpandArgs a{ctx->scene, ctx->b_in.as<double>(), ctx->b_push.as<double>(), ctx->b_out.as<double>(),
               ctx->b_status.as<int32_t>(), ctx->b_a.as<uint8_t>(), ctx->b_e.as<int32_t>(), ctx->b_b.as<double>(), P};
  if (use_warp(ctx, ctx->scene_all_discs, n, P, true)) {
    PPG_WARP_LAUNCH(expand_warp_kernel, !ctx->scene_all_discs, n, P, st, C, a);
  } else if (use_disc(ctx, ctx->scene_all_discs, n)) {
    // child = parent, resolve in place on the register-resident kernel, then
    // sample + grasp (or restore the parent for a failed simulation)
    CK(cudaMemcpyAsync(ctx->b_out.p, ctx->b_in.p, pbytes, cudaMemcpyDeviceToDevice, st));
    ResolveArgs ra{ctx->scene, ctx->b_out.as<double>(), ctx->b_push.as<double>(), ctx->b_out.as<double>(),
                   ctx->b_status.as<int32_t>(), nullptr, nullptr, P};
    const int rc = launch_disc(ctx, C, ra, n, P, st);
    if (rc != PPG_SUCCESS) return rc;
    expand_post_kernel<<<(P + kBlock - 1) / kBlock, kBlock, smem_for(n), st>>>(C, a);
  } else {
    expand_kernel<<<(P + kBlock - 1) / kBlock, kBlock, smem_for(n), st>>>(C, a);
  }
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(child_poses, ctx->b_out.p, pbytes, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(status, ctx->b_status.p, static_cast<size_t>(P) * 4, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(graspable, ctx->b_a.p, P, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(n_untried, ctx->b_e.p, static_cast<size_t>(P) * 4, cudaMemcpyDeviceToHost, st));
  if (untried) CK(cudaMemcpyAsync(untried, ctx->b_b.p, ubytes, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return PPG_SUCCESS;
}

}  // extern "C"

// ---- lockstep engine (pmbs.cpp:133-234) host side --------------------------

// Allocates and initialises the lockstep state for `used` local environments
// (global indices env_lo .. env_lo+used-1 of a batch of used_global) over the
// given nodes; runs lock_init_kernel.
int lock_setup(ppg_ctx* ctx, const double* node_poses, const int32_t* node_meta, int n_nodes, int used,
                      int used_global, int env_lo, int leaf_parallel, uint64_t seed, uint64_t iteration,
                      int depth_cap) {
  cudaStream_t st = ctx->stream;
  const int n = ctx->scene.n;
  const int E = used > 0 ? used : 1;
  CK(ctx->l_node.ensure(static_cast<size_t>(E) * 4));
  CK(ctx->l_pushes.ensure(static_cast<size_t>(E) * 4));
  CK(ctx->l_done.ensure(E));
  CK(ctx->l_byg.ensure(E));
  CK(ctx->l_harv.ensure(E));
  CK(ctx->l_flag.ensure(E));
  CK(ctx->l_reward.ensure(static_cast<size_t>(E) * 8));
  CK(ctx->l_poses.ensure(static_cast<size_t>(E) * 3 * n * 8));
  CK(ctx->l_mt.ensure(static_cast<size_t>(E) * 312 * 8));
  CK(ctx->l_mtidx.ensure(static_cast<size_t>(E) * 4));
  CK(ctx->l_W.ensure(static_cast<size_t>(n_nodes) * 4));
  CK(ctx->l_rew.ensure(static_cast<size_t>(n_nodes) * 8));
  CK(ctx->l_active.ensure(static_cast<size_t>(E) * 4));
  CK(ctx->l_nactive.ensure(16));
  CK(ctx->l_counters.ensure(4 * 8));
  CK(ctx->l_npose.ensure(static_cast<size_t>(n_nodes) * n * 3 * 8));
  CK(ctx->l_nmeta.ensure(static_cast<size_t>(n_nodes) * 3 * 4));
  CK(ctx->l_push.ensure(static_cast<size_t>(E) * 32));
  CK(ctx->l_status.ensure(static_cast<size_t>(E) * 4));
  CK(ctx->l_stepping.ensure(static_cast<size_t>(E) * 4 + 16));
  CK(ctx->l_rec.ensure(static_cast<size_t>(E) * (4 + 4 + 1 + 8) + 64));
  CK(ctx->l_around.ensure(static_cast<size_t>(E) * 4));
  CK(ctx->l_astate.ensure(static_cast<size_t>(E) * 4));
  CK(ctx->l_aW.ensure(static_cast<size_t>(kAsyncK) * n_nodes * 4));
  CK(ctx->l_aP.ensure(static_cast<size_t>(kAsyncK) * n_nodes * 4));
  CK(ctx->l_spec.ensure(static_cast<size_t>(E) * 16 + 16));
  CK(ctx->l_actr.ensure(static_cast<size_t>(kAsyncK) * kRingCtr * 4));
  CK(ctx->l_adl.ensure(static_cast<size_t>(kAsyncK) * E * 4));
  CK(ctx->l_actl.ensure(64));
  CK(cudaMemsetAsync(ctx->l_actl.p, 0, 64, st));
  CK(ctx->l_fin.ensure(static_cast<size_t>(E) * 4 + 16));
  CK(ctx->l_rsi.ensure(static_cast<size_t>(E) * 4));
  CK(ctx->l_ract.ensure(static_cast<size_t>(E) * 4));
  CK(cudaMemcpyAsync(ctx->l_npose.p, node_poses, static_cast<size_t>(n_nodes) * n * 3 * 8, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(ctx->l_nmeta.p, node_meta, static_cast<size_t>(n_nodes) * 3 * 4, cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(ctx->l_counters.p, 0, 32, st));
  ctx->lc = make_const(ctx->params, n, ctx->side, ctx->margin);
  LockArgs& a = ctx->la;
  a = LockArgs{};
  a.S = ctx->scene;
  a.node_poses = ctx->l_npose.as<double>();
  a.node_meta = ctx->l_nmeta.as<int32_t>();
  a.n_nodes = n_nodes;
  a.used = used;
  a.used_global = used_global;
  a.env_lo = env_lo;
  a.leaf_parallel = leaf_parallel;
  a.cap = depth_cap;
  a.seed = seed;
  a.iteration = iteration;
  a.env_node = ctx->l_node.as<int32_t>();
  a.env_pushes = ctx->l_pushes.as<int32_t>();
  a.env_done = ctx->l_done.as<uint8_t>();
  a.env_bygrasp = ctx->l_byg.as<uint8_t>();
  a.env_harvested = ctx->l_harv.as<uint8_t>();
  a.env_flag = ctx->l_flag.as<uint8_t>();
  a.env_reward = ctx->l_reward.as<double>();
  a.env_poses = ctx->l_poses.as<double>();
  a.mt = ctx->l_mt.as<uint64_t>();
  a.mt_idx = ctx->l_mtidx.as<int32_t>();
  a.E = E;
  a.W = ctx->l_W.as<int32_t>();
  a.rew = ctx->l_rew.as<unsigned long long>();
  a.active = ctx->l_active.as<int32_t>();
  a.n_active = ctx->l_nactive.as<int32_t>();
  a.counters = ctx->l_counters.as<long long>();
  a.env_push = ctx->l_push.as<double>();
  a.env_status = ctx->l_status.as<int32_t>();
  a.n_stepping = ctx->l_stepping.as<int32_t>();
  a.stepping = ctx->l_stepping.as<int32_t>() + 4;
  {
    char* r = ctx->l_rec.as<char>();
    a.n_rec = reinterpret_cast<int32_t*>(r);
    a.rec_env = reinterpret_cast<int32_t*>(r + 16);
    a.rec_node = a.rec_env + E;
    a.rec_reward = reinterpret_cast<double*>(r + 16 + static_cast<size_t>(E) * 8 + 8 - ((16 + E * 8) % 8));
    a.rec_grasp = reinterpret_cast<uint8_t*>(a.rec_reward + E);
  }
  a.env_round = ctx->l_around.as<int32_t>();
  a.env_state = ctx->l_astate.as<int32_t>();
  a.a_W = ctx->l_aW.as<int32_t>();
  a.a_P = ctx->l_aP.as<int32_t>();
  a.a_spec = speculate_enabled() && E <= kSpecMaxEnvs ? ctx->l_spec.as<int4>() : nullptr;
  a.a_ctr = ctx->l_actr.as<int32_t>();
  a.a_dl = ctx->l_adl.as<int32_t>();
  a.a_ctl = ctx->l_actl.as<int32_t>();
  a.a_wcap = n_nodes;
  a.fin_count = ctx->l_fin.as<int32_t>();
  a.fin_list = ctx->l_fin.as<int32_t>() + 4;
  a.resume_si = ctx->l_rsi.as<int32_t>();
  a.resume_active = ctx->l_ract.as<uint32_t>();
  ctx->lra = ResolveArgs{ctx->scene, a.env_poses, a.env_push, a.env_poses, a.env_status, nullptr, nullptr, 0};
  ctx->lra.idx = a.stepping;
  ctx->lra.E_dev = a.n_stepping;
  const int ginit = ((E > n_nodes ? E : n_nodes) + 255) / 256;
  lock_init_kernel<<<ginit, 256, 0, st>>>(ctx->lc, a);
  CK(cudaGetLastError());
  return PPG_SUCCESS;
}

// One lockstep round over the current active list (at most `act` envs):
// latency mode (one warp per env), the 3-phase disc pipeline, or the generic
// one-lane step.
int lock_round(ppg_ctx* ctx, int act) {
  return lock_round_on(ctx, ctx->lc, ctx->la, ctx->lra, act, round_mode(ctx, ctx->scene.n, act), ctx->stream);
}

int lock_check(ppg_ctx* ctx, int n_nodes, int n_envs, int depth_cap) {
  if (n_envs < n_nodes) {
    ctx->err = "lockstep_simulate: fewer environments than nodes";
    return PPG_EINVAL;
  }
  if (!ctx->has_scene) {
    ctx->err = "no scene installed";
    return PPG_EINVAL;
  }
  if (depth_cap + 1 >= kMaxGammaPow) {
    ctx->err = "depth cap too large";
    return PPG_EINVAL;
  }
  return PPG_SUCCESS;
}

unsigned long long* step_trace_buffer(ppg_ctx* ctx) {
  static const char* path = std::getenv("PPG_STEP_TRACE");
  if (!path) return nullptr;
  constexpr unsigned long long kRecs = 1ull << 22;
  if (ctx->trace_buf.cap == 0) {
    if (ctx->trace_buf.ensure((2 + 4 * kRecs) * 8) != cudaSuccess) return nullptr;
    const unsigned long long hdr[2] = {0ull, kRecs};
    cudaMemcpy(ctx->trace_buf.p, hdr, 16, cudaMemcpyHostToDevice);
  }
  return ctx->trace_buf.as<unsigned long long>();
}

void step_trace_dump(ppg_ctx* ctx) {
  static const char* path = std::getenv("PPG_STEP_TRACE");
  if (!path || ctx->trace_buf.cap == 0) return;
  cudaStreamSynchronize(ctx->stream);
  unsigned long long hdr[2];
  cudaMemcpy(hdr, ctx->trace_buf.p, 16, cudaMemcpyDeviceToHost);
  const unsigned long long k = hdr[0] < hdr[1] ? hdr[0] : hdr[1];
  std::vector<unsigned long long> rec(4 * k);
  if (k) cudaMemcpy(rec.data(), ctx->trace_buf.as<unsigned long long>() + 2, 32 * k, cudaMemcpyDeviceToHost);
  if (FILE* f = std::fopen(path, "ab")) {
    const unsigned long long marker = ~0ull;  // one call per block of records
    std::fwrite(&marker, 8, 1, f);
    std::fwrite(&k, 8, 1, f);
    std::fwrite(rec.data(), 32, k, f);
    std::fclose(f);
  }
  const unsigned long long zero = 0;
  cudaMemcpy(ctx->trace_buf.p, &zero, 8, cudaMemcpyHostToDevice);
}

extern "C" {

int ppg_simulate(ppg_ctx* ctx, const double* node_poses, const int32_t* node_meta, int n_nodes, int n_envs,
                 int leaf_parallel, uint64_t seed, uint64_t iteration, int depth_cap, double* rewards_out,
                 int64_t* counters) {
  if (!ctx) return PPG_EINVAL;
  if (n_nodes <= 0) return PPG_SUCCESS;
  if (ctx->group)  // multi-GPU: the rollout batch sharded by environment (multi.cu)
    return ppg::simulate_sharded(ctx, node_poses, node_meta, n_nodes, n_envs, leaf_parallel, seed, iteration,
                                 depth_cap, rewards_out, counters);
  int rc = lock_check(ctx, n_nodes, n_envs, depth_cap);
  if (rc != PPG_SUCCESS) return rc;
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  const int used = leaf_parallel ? n_envs : n_nodes;
  rc = lock_setup(ctx, node_poses, node_meta, n_nodes, used, used, 0, leaf_parallel, seed, iteration, depth_cap);
  if (rc != PPG_SUCCESS) return rc;
  ctx->la.step_trace = step_trace_buffer(ctx);
  // PPG_ROUND_TRACE=1: per-round active count, mode and device time to stderr (experiments)
  static const bool trace = std::getenv("PPG_ROUND_TRACE") != nullptr;
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  if (trace) {
    cudaEventCreate(&t0);
    cudaEventCreate(&t1);
  }
  for (int round = 0;; ++round) {
    lock_harvest_kernel<<<1, 1024, 0, st>>>(ctx->lc, ctx->la);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(ctx->h_nactive, ctx->la.n_active, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const int act = *ctx->h_nactive;
    if (act == 0) break;
    if (trace) cudaEventRecord(t0, st);
    if (round == 0 && wave_enabled(ctx) && round_mode(ctx, ctx->scene.n, act) == RoundMode::kHybrid) {
      // large disc batch: wave rounds while the batch is wide, then the
      // asynchronous kernel for the tail (warp_env.cu)
      int32_t* ctl = ctx->la.a_ctl;
      const int32_t one = 1;
      CK(cudaMemcpyAsync(ctl + 6, &one, 4, cudaMemcpyHostToDevice, st));  // round_mode word: waves
      LockArgs wa = ctx->la;
      wa.round_mode = ctl + 6;
      wa.go = ctl + 7;
      wa.wave_switch = ctx->wave_switch;
      wa.wave_budget = ctx->wave_budget;
      if (trace) cudaEventRecord(t0, st);
      for (int wave = 0;; ++wave) {
        rc = launch_wave(ctx, ctx->lc, wa, ctx->lra, used, st);
        if (rc != PPG_SUCCESS) return rc;
        int32_t hctl[16];
        CK(cudaMemcpyAsync(hctl, ctl, 64, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (trace) {
          cudaEventRecord(t1, st);
          cudaEventSynchronize(t1);
          float ms = 0.f;
          cudaEventElapsedTime(&ms, t0, t1);
          std::fprintf(stderr, "wave %d H %d gone %d switch %d ms %.4f\n", wave, hctl[0], hctl[2], hctl[5], ms);
          cudaEventRecord(t0, st);
        }
        if (hctl[7] == 0) break;  // every env done and harvested
        if (hctl[5] == 2) {       // the hand-over wave ran: the asynchronous kernel finishes the call
          rc = launch_async(ctx, ctx->lc, wa, used, st, true);
          if (rc != PPG_SUCCESS) return rc;
          CK(cudaMemcpyAsync(hctl, ctl, 16, cudaMemcpyDeviceToHost, st));
          CK(cudaStreamSynchronize(st));
          if (trace) {
            cudaEventRecord(t1, st);
            cudaEventSynchronize(t1);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, t0, t1);
            std::fprintf(stderr, "async tail from H %d: complete round %d ms %.4f\n", wa.wave_switch, hctl[0], ms);
          }
          if (hctl[3] != 0) {
            ctx->err = "asynchronous lockstep stalled (protocol error)";
            return PPG_ECUDA;
          }
          break;
        }
        if (wave > kLockRoundLimit) {
          ctx->err = "wave rounds did not terminate";
          return PPG_EINVAL;
        }
      }
      break;
    }
    const bool go_async = async_enabled(ctx) && round_mode(ctx, ctx->scene.n, act) == RoundMode::kWarp;
    if (go_async) {  // every remaining round, barrier-free (warp_env.cu lock_async_kernel)
      rc = launch_async(ctx, ctx->lc, ctx->la, used, st, false);
      if (rc != PPG_SUCCESS) return rc;
      int32_t ctl[4];
      CK(cudaMemcpyAsync(ctl, ctx->la.a_ctl, 16, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      if (ctl[3] != 0) {
        ctx->err = "asynchronous lockstep stalled (protocol error)";
        return PPG_ECUDA;
      }
    } else {
      rc = lock_round(ctx, act);
      if (rc != PPG_SUCCESS) return rc;
    }
    if (trace) {
      cudaEventRecord(t1, st);
      cudaEventSynchronize(t1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, t0, t1);
      std::fprintf(stderr, "round %d active %d mode %d ms %.4f\n", round, act,
                   static_cast<int>(round_mode(ctx, ctx->scene.n, act)), ms);
    }
  }
  if (trace) {
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
  }
  CK(cudaMemcpyAsync(rewards_out, ctx->la.rew, static_cast<size_t>(n_nodes) * 8, cudaMemcpyDeviceToHost, st));
  if (counters) CK(cudaMemcpyAsync(counters, ctx->la.counters, 32, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (ctx->la.step_trace) step_trace_dump(ctx);
  return PPG_SUCCESS;
}

int ppg_simulate_count(ppg_ctx* ctx, const double* node_poses, const int32_t* node_meta, int n_nodes, int n_envs,
                       int leaf_parallel, uint64_t seed, uint64_t iteration, int depth_cap, int64_t* ops_out,
                       int64_t* counters) {
  if (!ctx || !ops_out) return PPG_EINVAL;
  if (n_nodes <= 0) return PPG_SUCCESS;
  int rc = lock_check(ctx, n_nodes, n_envs, depth_cap);
  if (rc != PPG_SUCCESS) return rc;
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  const int used = leaf_parallel ? n_envs : n_nodes;
  rc = lock_setup(ctx, node_poses, node_meta, n_nodes, used, used, 0, leaf_parallel, seed, iteration, depth_cap);
  if (rc != PPG_SUCCESS) return rc;
  CK(ctx->b_e.ensure(64));
  unsigned long long* ops = ctx->b_e.as<unsigned long long>();
  CK(cudaMemsetAsync(ops, 0, 24, st));
  const int n = ctx->scene.n;
  for (;;) {
    lock_harvest_kernel<<<1, 1024, 0, st>>>(ctx->lc, ctx->la);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(ctx->h_nactive, ctx->la.n_active, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const int act = *ctx->h_nactive;
    if (act == 0) break;
    lock_step_count_kernel<<<(act + kBlock - 1) / kBlock, kBlock, smem_for(n), st>>>(ctx->lc, ctx->la, ops);
    CK(cudaGetLastError());
  }
  CK(cudaMemcpyAsync(ops_out, ops, 24, cudaMemcpyDeviceToHost, st));
  if (counters) CK(cudaMemcpyAsync(counters, ctx->la.counters, 32, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return PPG_SUCCESS;
}

int ppg_lock_begin(ppg_ctx* ctx, const double* node_poses, const int32_t* node_meta, int n_nodes, int used_envs,
                   int env_lo, int env_hi, int leaf_parallel, uint64_t seed, uint64_t iteration, int depth_cap) {
  if (!ctx || n_nodes <= 0 || env_lo < 0 || env_hi < env_lo || env_hi > used_envs) return PPG_EINVAL;
  int rc = lock_check(ctx, n_nodes, leaf_parallel ? used_envs : n_nodes, depth_cap);
  if (rc != PPG_SUCCESS) return rc;
  CK(cudaSetDevice(ctx->device));
  rc = lock_setup(ctx, node_poses, node_meta, n_nodes, env_hi - env_lo, used_envs, env_lo, leaf_parallel, seed,
                  iteration, depth_cap);
  if (rc != PPG_SUCCESS) return rc;
  ctx->lock_active_hint = env_hi - env_lo;
  return PPG_SUCCESS;
}

int ppg_lock_report(ppg_ctx* ctx, int32_t* rec_env, int32_t* rec_node, uint8_t* rec_grasp, double* rec_reward,
                    int32_t* n_rec, int32_t* w_local, int32_t* n_active) {
  if (!ctx) return PPG_EINVAL;
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  LockArgs& a = ctx->la;
  lock_report_kernel<<<1, 1024, 0, st>>>(ctx->lc, a);
  CK(cudaGetLastError());
  int32_t hdr[2];
  CK(cudaMemcpyAsync(&hdr[0], a.n_rec, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&hdr[1], a.n_active, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(w_local, a.W, static_cast<size_t>(a.n_nodes) * 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const int k = hdr[0];
  if (k > 0) {
    CK(cudaMemcpyAsync(rec_env, a.rec_env, static_cast<size_t>(k) * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(rec_node, a.rec_node, static_cast<size_t>(k) * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(rec_grasp, a.rec_grasp, static_cast<size_t>(k), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(rec_reward, a.rec_reward, static_cast<size_t>(k) * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  *n_rec = k;
  *n_active = hdr[1];
  ctx->lock_active_hint = hdr[1];
  return PPG_SUCCESS;
}

int ppg_lock_repurpose(ppg_ctx* ctx, const int32_t* env, const int32_t* node, int count) {
  if (!ctx || count < 0) return PPG_EINVAL;
  if (count == 0) return PPG_SUCCESS;
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  CK(ctx->b_d.ensure(static_cast<size_t>(count) * 8));
  int32_t* d = ctx->b_d.as<int32_t>();
  CK(cudaMemcpyAsync(d, env, static_cast<size_t>(count) * 4, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d + count, node, static_cast<size_t>(count) * 4, cudaMemcpyHostToDevice, st));
  lock_repurpose_kernel<<<(count + 255) / 256, 256, 0, st>>>(ctx->lc, ctx->la, d, d + count, count);
  CK(cudaGetLastError());
  ctx->lock_active_hint += count;
  return PPG_SUCCESS;
}

int ppg_lock_step(ppg_ctx* ctx) {
  if (!ctx) return PPG_EINVAL;
  CK(cudaSetDevice(ctx->device));
  if (ctx->lock_active_hint <= 0) return PPG_SUCCESS;
  const int rc = lock_round(ctx, ctx->lock_active_hint);
  if (rc != PPG_SUCCESS) return rc;
  CK(cudaStreamSynchronize(ctx->stream));
  return PPG_SUCCESS;
}

int ppg_set_planner(ppg_ctx* ctx, int mode) {
  if (!ctx || mode < PPG_PLANNER_AUTO || mode > PPG_PLANNER_DEVICE) return PPG_EINVAL;
  ctx->planner = mode;
  return PPG_SUCCESS;
}

int ppg_set_simulate_hook(ppg_ctx* ctx, ppg_simulate_fn fn, void* user) {
  if (!ctx) return PPG_EINVAL;
  ctx->sim_hook = fn;
  ctx->sim_hook_user = user;
  return PPG_SUCCESS;
}

int ppg_lock_counters(ppg_ctx* ctx, int64_t* counters) {
  if (!ctx || !counters) return PPG_EINVAL;
  CK(cudaSetDevice(ctx->device));
  CK(cudaMemcpyAsync(counters, ctx->la.counters, 32, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return PPG_SUCCESS;
}

int ppg_debug_sincos(ppg_ctx* ctx, const double* x, int n, double* s, double* c) {
  if (!ctx || n < 0) return PPG_EINVAL;
  if (n == 0) return PPG_SUCCESS;
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  const size_t b = static_cast<size_t>(n) * 8;
  CK(ctx->b_a.ensure(b));
  CK(ctx->b_b.ensure(b));
  CK(ctx->b_c.ensure(b));
  CK(cudaMemcpyAsync(ctx->b_a.p, x, b, cudaMemcpyHostToDevice, st));
  debug_sincos_kernel<<<(n + 255) / 256, 256, 0, st>>>(ctx->b_a.as<double>(), n, ctx->b_b.as<double>(),
                                                       ctx->b_c.as<double>());
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(s, ctx->b_b.p, b, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(c, ctx->b_c.p, b, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return PPG_SUCCESS;
}

int ppg_measure_fp64_peak(ppg_ctx* ctx, double* dfma_per_s, double* seconds) {
  if (!ctx || !dfma_per_s) return PPG_EINVAL;
  CK(cudaSetDevice(ctx->device));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
  const int blocks = sms * 8, threads = 256, iters = 1 << 16;
  CK(ctx->b_e.ensure(static_cast<size_t>(blocks) * 8));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  double best = 0.0, best_s = 0.0;
  for (int rep = 0; rep < 4; ++rep) {
    CK(cudaEventRecord(e0, ctx->stream));
    fp64_peak_kernel<<<blocks, threads, 0, ctx->stream>>>(ctx->b_e.as<double>(), iters, 0.999999, 1e-7);
    CK(cudaEventRecord(e1, ctx->stream));
    CK(cudaEventSynchronize(e1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double rate = static_cast<double>(blocks) * threads * 8.0 * iters / (ms * 1e-3);
    if (rate > best) {
      best = rate;
      best_s = ms * 1e-3;
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *dfma_per_s = best;
  if (seconds) *seconds = best_s;
  return PPG_SUCCESS;
}

int ppg_state_digest(const ppg_shapes* sh, const double* poses, int E, uint64_t* out) {
  if (!sh || !poses || !out) return PPG_EINVAL;
  const int n = sh->n_objects;
  for (int e = 0; e < E; ++e) {
    const int t = sh->n_tables == 1 ? 0 : e;
    uint64_t h = 1469598103934665603ull;
    auto mix = [&h](const void* data, size_t len) {
      const unsigned char* p = static_cast<const unsigned char*>(data);
      for (size_t i = 0; i < len; ++i) {
        h ^= p[i];
        h *= 1099511628211ull;
      }
    };
    const int32_t tgt = sh->target_index[t];
    mix(&tgt, 4);
    mix(&sh->side_length, 8);
    for (int i = 0; i < n; ++i) {
      const int32_t kind = sh->kind[t * n + i];
      mix(&kind, 4);
      mix(&sh->radius[t * n + i], 8);
      if (kind != PPG_DISC && sh->n_vertices && sh->vertices)
        for (int k = 0; k < sh->n_vertices[t * n + i]; ++k)
          mix(&sh->vertices[((static_cast<size_t>(t) * n + i) * kMaxV + k) * 2], 16);
      mix(&poses[(static_cast<size_t>(e) * n + i) * 3], 24);
    }
    out[e] = h;
  }
  return PPG_SUCCESS;
}

}  // extern "C"

// internal accessors for planner.cpp
namespace ppg {
const ppg_params& ctx_params(const ppg_ctx* ctx) { return ctx->params; }
SimHook ctx_sim_hook(const ppg_ctx* ctx) { return SimHook{ctx->sim_hook, ctx->sim_hook_user}; }
int ctx_planner(const ppg_ctx* ctx) { return ctx->planner; }
int ctx_n_objects(const ppg_ctx* ctx) { return ctx->has_scene ? ctx->scene.n : 0; }
void ctx_set_error(ppg_ctx* ctx, const char* msg) { ctx->err = msg; }
}  // namespace ppg
