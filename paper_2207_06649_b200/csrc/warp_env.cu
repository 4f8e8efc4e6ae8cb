// warp_env.cu — latency mode kernels (helpers in warp_env.cuh): ONE WARP PER ENVIRONMENT (disc scenes, n <= 23).
//
// The lane-per-env kernels (resolve_disc.cu) maximise throughput when there
// are many more environments than lanes; a PMBS search at the reference
// defaults (N_e = 64, 25-40 % of envs active per lockstep round) has a few
// dozen to a few thousand environments per launch, and there the latency of
// one sequential environment is what a round costs.  Here the 32 lanes of a
// warp cooperate on one environment, bit-exactly:
//
//  * tip phase (push_sim.cpp:90-100): lane i owns object i — objects are
//    independent in the tip loop;
//  * pair broad phase (push_sim.cpp:107-108): pair p is tested by lane p % 32,
//    candidates collected with __ballot_sync into warp-uniform masks;
//  * pair narrow phase: the candidates are processed in lexicographic order
//    by the whole warp (identical values in every lane); after a hit on (i,j)
//    the lanes owning LATER pairs touching i or j re-test them on the new
//    poses, so every set bit always means "passes the broad test now" —
//    exactly the reference's in-place Gauss-Seidel sweep (push_sim.cpp:101-117);
//  * the convergence test max_pen <= eps (push_sim.cpp:119) is a ballot;
//  * sample_pushes (actions.cpp:51-73): candidate c tested by lane c % 32,
//    validity ballots give the (object, angle)-ordered list;
//  * graspable (actions.cpp:113-147): lane k evaluates grasp angle k; the
//    first strict maximum in index order == max margin, lowest k on ties;
//  * MT19937-64: the 312-word block twist runs on 32 lanes in its three
//    dependency phases (libstdc++ _M_gen_rand).
//
// Poses live in shared memory (per-warp block x[32] | y[32] | theta[32] |
// r[32]); every max reduction is over non-negative values starting at +0.0,
// so its result does not depend on the order.
#include <cuda_runtime.h>

#include "warp_env.cuh"
#include "warp_poly.cuh"
#include "pushplan_gpu.h"  // status codes of the debug accessor

namespace ppg {

#ifdef PPG_PHASE_TRACE_BUILD
// latency split of the asynchronous kernel's env-steps (experiments; build
// with EXTRA_NVFLAGS=-DPPG_PHASE_TRACE_BUILD): globaltimer ns summed over
// steps — [0] sample, [1] pick, [2] resolve, [3] graspable + bookkeeping,
// [4] steps
__device__ unsigned long long g_phase_ns[8];
__device__ unsigned long long g_await_t0[65536];  // [5] / [6]: AWAIT wait ns / count
#define PPG_PHASE_MARK(slot, t_prev)                                          \
  do {                                                                        \
    if (l == 0) {                                                             \
      unsigned long long t_now;                                               \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_now));               \
      atomicAdd(&g_phase_ns[slot], t_now - t_prev);                           \
      t_prev = t_now;                                                         \
    }                                                                         \
  } while (0)
#endif

// ---------------------------------------------------------------------------

// batch_resolve, one warp per environment (small batches).
// Polygon caches of the latency-mode kernels (kPoly instantiations only).
#define PPG_POLY_SMEM                                      \
  __shared__ V2 poly_wv[kPoly ? kWarpsPerBlock : 1][kPoly ? kPolyMaxN * kMaxV : 1]; \
  __shared__ V2 poly_cen[kPoly ? kWarpsPerBlock : 1][kPoly ? kPolyMaxN : 1];

// resolve with the variant for the scene's object kinds (warp_poly.cuh for
// scenes with polygons)
template <int NW, bool kPoly>
PPG_DI int warp_resolve_any(WarpEnv& W, const WarpPoly& G, const PolyShape& O, const ShapeView& S, const SimConst& C,
                            const uint16_t* pij, V2 start, V2 end, bool check_start, double* residual) {
  if constexpr (kPoly) {
    return warp_resolve_poly<NW>(W, G, O, S, C, pij, start, end, check_start, residual);
  } else {
    return warp_resolve<NW>(W, C, pij, start, end, check_start, residual);
  }
}

// Pose load of the latency-mode kernels: for polygon scenes also the trig
// planes and the world-polygon caches, which the sampler / graspable helpers
// (world_polygon on the PoseView) and warp_resolve_poly read.
template <bool kPoly>
PPG_DI PolyShape warp_load_any(WarpEnv& W, const WarpPoly& G, const double* poses, const ShapeView& S) {
  warp_load(W, poses, S);
  PolyShape O{0, 0, 0.0, 0.0};
  if constexpr (kPoly) O = warp_poly_load(W, G, S);
  return O;
}

template <int NW, bool kPoly>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, kPoly ? 4 : 1) resolve_warp_kernel(const __grid_constant__ SimConst C,
                                                                          ResolveArgs a) {
  __shared__ double blk[kWarpsPerBlock][160];
  PPG_POLY_SMEM
  __shared__ uint16_t pij[kWarpMaxN * (kWarpMaxN - 1) / 2];
  build_pairs(pij, C.n);
  const int wib = threadIdx.x >> 5;
  const int E = a.E_dev ? *a.E_dev : a.E;
  const int n = C.n;
  const WarpPoly G{poly_wv[kPoly ? wib : 0], poly_cen[kPoly ? wib : 0]};
  // one env per warp; with a work counter the warps are persistent and take
  // the next env when done (envs differ widely in cost)
  for (int e = blockIdx.x * kWarpsPerBlock + wib; e < E;) {
    const int ee = a.idx ? a.idx[e] : e;
    WarpEnv W(blk[wib], n, static_cast<int>(threadIdx.x & 31));
    const ShapeView S = a.S.view(a.S.T == 1 ? 0 : ee);
    const PolyShape O = warp_load_any<kPoly>(W, G, a.poses_in + static_cast<size_t>(ee) * n * 3, S);
    const double* pu = a.pushes + static_cast<size_t>(ee) * 4;
    double residual = 0.0;
    const int st = warp_resolve_any<NW, kPoly>(W, G, O, S, C, pij, V2{pu[0], pu[1]}, V2{pu[2], pu[3]}, true,
                                               &residual);
    if (W.lane == 0) {
      a.status[ee] = st;
      if (a.residual) a.residual[ee] = residual;
    }
    double* out = a.poses_out + static_cast<size_t>(ee) * n * 3;
    if (st == 0) {
      warp_store(W, out);
    } else {
      for (int i = W.lane; i < n * 3; i += 32) out[i] = 0.0;
    }
    if (!a.work_counter) break;
    int nx = 0;
    if (W.lane == 0) nx = atomicAdd(a.work_counter, 1);
    e = gridDim.x * kWarpsPerBlock + __shfl_sync(kFull, nx, 0);
    __syncwarp();  // the warp's shared blocks are reused by the next env
  }
}

// sample_pushes (actions.cpp:51-73: the full ordered candidate list) and /
// or graspable (actions.cpp:113-147) of E states, one warp per state: the
// candidates' validity tests and the 16 grasp angles run across the lanes
// (the one-lane kernels walk them in sequence: ~0.26 ms for one state).
template <bool kPoly>
__global__ void __launch_bounds__(kWarpsPerBlock * 32) sample_grasp_warp_kernel(const __grid_constant__ SimConst C,
                                                                               SampleArgs a) {
  __shared__ double blk[kWarpsPerBlock][160];
  PPG_POLY_SMEM
  __shared__ unsigned valid[kWarpsPerBlock][32];
  const int wib = threadIdx.x >> 5;
  const int e = blockIdx.x * kWarpsPerBlock + wib;
  if (e >= a.E) return;
  const int n = C.n, l = threadIdx.x & 31;
  const int t = a.S.T == 1 ? 0 : e;
  const ShapeView S = a.S.view(t);
  WarpEnv W(blk[wib], n, l);
  const WarpPoly G{poly_wv[kPoly ? wib : 0], poly_cen[kPoly ? wib : 0]};
  warp_load_any<kPoly>(W, G, a.poses + static_cast<size_t>(e) * n * 3, S);
  if (a.out) {
    const int count = warp_sample_mask(W, S, C, valid[wib]);
    const int nw = (n * C.na + 31) >> 5;
    double* out = a.out + static_cast<size_t>(e) * n * C.na * 4;
    const PoseView PV = W.view();
    int base = 0;
    for (int w = 0; w < nw; ++w) {
      const unsigned b = valid[wib][w];
      if (b >> l & 1u) {
        const int c = 32 * w + l;
        V2 s0, t0;
        push_candidate(PV, S, C, c / C.na, c % C.na, false, s0, t0);
        double* q = out + static_cast<size_t>(base + __popc(b & ((1u << l) - 1u))) * 4;
        q[0] = s0.x;
        q[1] = s0.y;
        q[2] = t0.x;
        q[3] = t0.y;
      }
      base += __popc(b);
    }
    if (l == 0) a.count[e] = count;
  }
  if (a.grasp) {
    const GraspOut g = warp_graspable(W, S, C, a.S.target[t]);
    if (l == 0) {
      a.grasp[e] = g.graspable ? 1 : 0;
      a.margin[e] = g.margin;
      a.bx[e] = g.x;
      a.by[e] = g.y;
      a.bk[e] = g.k;
    }
  }
}
template __global__ void sample_grasp_warp_kernel<false>(const __grid_constant__ SimConst, SampleArgs);
template __global__ void sample_grasp_warp_kernel<true>(const __grid_constant__ SimConst, SampleArgs);

// batch_expand prepare (pmbs.cpp:82-93), one warp per (node, action) pair.
template <int NW, bool kPoly>
__global__ void __launch_bounds__(kWarpsPerBlock * 32) expand_warp_kernel(const __grid_constant__ SimConst C,
                                                                         ExpandArgs a) {
  __shared__ double blk[kWarpsPerBlock][160];
  PPG_POLY_SMEM
  __shared__ unsigned valid[kWarpsPerBlock][32];
  __shared__ uint16_t pij[kWarpMaxN * (kWarpMaxN - 1) / 2];
  build_pairs(pij, C.n);
  const int wib = threadIdx.x >> 5;
  const int p = blockIdx.x * kWarpsPerBlock + wib;
  if (p >= (a.P_dev ? *a.P_dev : a.P)) return;
  const int n = C.n, l = threadIdx.x & 31;
  WarpEnv W(blk[wib], n, l);
  const ShapeView S = a.S.view(0);
  const double* parent = a.parent_poses + static_cast<size_t>(p) * n * 3;
  const WarpPoly G{poly_wv[kPoly ? wib : 0], poly_cen[kPoly ? wib : 0]};
  const PolyShape O = warp_load_any<kPoly>(W, G, parent, S);
  const double* act = a.actions + static_cast<size_t>(p) * 4;
  double residual;
  const int st = warp_resolve_any<NW, kPoly>(W, G, O, S, C, pij, V2{act[0], act[1]}, V2{act[2], act[3]}, true,
                                             &residual);
  double* child = a.child_poses + static_cast<size_t>(p) * n * 3;
  if (l == 0) a.status[p] = st;
  if (st != 0) {  // dead child: copy of the parent state (mcts.cpp:89-92)
    for (int i = l; i < n * 3; i += 32) child[i] = parent[i];
    if (l == 0) {
      a.grasp[p] = 0;
      a.n_untried[p] = 0;
    }
    return;
  }
  warp_store(W, child);
  // full ordered untried list (sample_pushes, actions.cpp:51-73)
  const int count = warp_sample_mask(W, S, C, valid[wib]);
  const int total = n * C.na;
  const int nw = (total + 31) >> 5;
  double* out = a.untried + static_cast<size_t>(p) * n * C.na * 4;
  int base = 0;
  const PoseView PV = W.view();
  for (int w = 0; w < nw; ++w) {
    const unsigned b = valid[wib][w];
    if (b >> l & 1u) {
      const int c = 32 * w + l;
      V2 s, t;
      push_candidate(PV, S, C, c / C.na, c % C.na, false, s, t);
      double* q = out + static_cast<size_t>(base + __popc(b & ((1u << l) - 1u))) * 4;
      q[0] = s.x;
      q[1] = s.y;
      q[2] = t.x;
      q[3] = t.y;
    }
    base += __popc(b);
  }
  const GraspOut g = warp_graspable(W, S, C, a.S.target[0]);
  if (l == 0) {
    a.n_untried[p] = count;
    a.grasp[p] = g.graspable ? 1 : 0;
  }
}

// batch_expand prepare, hybrid (large batches of disc scenes): the pushes
// were resolved in place on the child buffer by the lane-per-env disc kernel;
// here one warp per (node, action) pair: dead child on failure, else the
// child's full untried list and grasp flag (pmbs.cpp:82-93; the tail of
// expand_warp_kernel).
template <bool kPoly>
__global__ void __launch_bounds__(kWarpsPerBlock * 32) expand_post_warp_kernel(const __grid_constant__ SimConst C,
                                                                              ExpandArgs a) {
  __shared__ double blk[kWarpsPerBlock][160];
  PPG_POLY_SMEM
  __shared__ unsigned valid[kWarpsPerBlock][32];
  const int wib = threadIdx.x >> 5;
  const int p = blockIdx.x * kWarpsPerBlock + wib;
  if (p >= (a.P_dev ? *a.P_dev : a.P)) return;
  const int n = C.n, l = threadIdx.x & 31;
  double* child = a.child_poses + static_cast<size_t>(p) * n * 3;
  if (a.status[p] != 0) {  // dead child: copy of the parent state (mcts.cpp:89-92)
    const double* parent = a.parent_poses + static_cast<size_t>(p) * n * 3;
    for (int i = l; i < n * 3; i += 32) child[i] = parent[i];
    if (l == 0) {
      a.grasp[p] = 0;
      a.n_untried[p] = 0;
    }
    return;
  }
  WarpEnv W(blk[wib], n, l);
  const ShapeView S = a.S.view(0);
  const WarpPoly G{poly_wv[kPoly ? wib : 0], poly_cen[kPoly ? wib : 0]};
  warp_load_any<kPoly>(W, G, child, S);
  const int count = warp_sample_mask(W, S, C, valid[wib]);
  const int nw = (n * C.na + 31) >> 5;
  double* out = a.untried + static_cast<size_t>(p) * n * C.na * 4;
  const PoseView PV = W.view();
  int base = 0;
  for (int w = 0; w < nw; ++w) {
    const unsigned b = valid[wib][w];
    if (b >> l & 1u) {
      const int c = 32 * w + l;
      V2 s0, t0;
      push_candidate(PV, S, C, c / C.na, c % C.na, false, s0, t0);
      double* q = out + static_cast<size_t>(base + __popc(b & ((1u << l) - 1u))) * 4;
      q[0] = s0.x;
      q[1] = s0.y;
      q[2] = t0.x;
      q[3] = t0.y;
    }
    base += __popc(b);
  }
  const GraspOut g = warp_graspable(W, S, C, a.S.target[0]);
  if (l == 0) {
    a.n_untried[p] = count;
    a.grasp[p] = g.graspable ? 1 : 0;
  }
}
template __global__ void expand_post_warp_kernel<false>(const __grid_constant__ SimConst, ExpandArgs);

// RolloutCursor::step (mcts.cpp:142-171) of env e by the calling warp:
// sample + pick + resolve + graspable, state in HBM (env_*), the warp's
// shared blocks `blk` / `valid` / the polygon caches as scratch.
template <int NW, bool kPoly>
PPG_DI int warp_rollout_step(const SimConst& C, const LockArgs& a, int e, double* blk, unsigned* valid,
                             const uint16_t* pij, const WarpPoly& G, bool frozen = false) {
  const int n = C.n, l = threadIdx.x & 31;
  WarpEnv W(blk, n, l);
  const ShapeView S = a.S.view(0);
  double* env = a.env_poses + static_cast<size_t>(e) * n * 3;
  const PolyShape O = warp_load_any<kPoly>(W, G, env, S);
  if (l == 0) atomicAdd(reinterpret_cast<unsigned long long*>(&a.counters[0]), 1ull);
#ifdef PPG_STEP_TRACE_BUILD  // per-step records for tools/async_model.py (build with EXTRA_NVFLAGS=-DPPG_STEP_TRACE_BUILD)
  unsigned long long t_start = 0;
  if (a.step_trace && l == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  struct TraceGuard {  // writes the record on every exit path
    const LockArgs& a;
    int e, l;
    unsigned long long t0;
    __device__ ~TraceGuard() {
      if (!a.step_trace || l != 0) return;
      unsigned long long t1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      const unsigned long long k = atomicAdd(a.step_trace, 1ull);
      if (k < a.step_trace[1]) {
        unsigned long long* r = a.step_trace + 2 + 4 * k;
        r[0] = static_cast<unsigned long long>(a.env_lo + e) | static_cast<unsigned long long>(a.counters[1]) << 32;
        r[1] = t0;
        r[2] = t1;
        r[3] = static_cast<unsigned long long>(a.env_done[e]) | static_cast<unsigned long long>(a.env_bygrasp[e]) << 1 |
               static_cast<unsigned long long>(a.env_node[e]) << 8 | (a.iteration & 0xffffffull) << 40;
      }
    }
  } trace_guard{a, e, l, t_start};
#endif
#ifdef PPG_PHASE_TRACE_BUILD
  unsigned long long t_ph = 0;
  if (l == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_ph));
  if (l == 0) atomicAdd(&g_phase_ns[4], 1ull);
#endif
  const int count = warp_sample_mask(W, S, C, valid);
#ifdef PPG_PHASE_TRACE_BUILD
  PPG_PHASE_MARK(0, t_ph);
#endif
  if (count == 0) {  // no legal push: reward 0 (mcts.cpp:146-150)
    if (l == 0) {
      a.env_done[e] = 1;
      a.env_reward[e] = 0.0;
    }
    return 0;
  }
  const MtView g{a.mt + e, a.E, frozen};
  int idx = a.mt_idx[e];
  const uint64_t k = warp_mt_pick(g, idx, static_cast<uint64_t>(count), l);
  if (l == 0) a.mt_idx[e] = idx;
  // k-th valid candidate in (object, angle) order
  int w = 0, seen = 0;
  while (seen + __popc(valid[w]) <= static_cast<int>(k)) seen += __popc(valid[w++]);
  unsigned bits = valid[w];
  for (int drop = static_cast<int>(k) - seen; drop > 0; --drop) bits &= bits - 1;
  const int c = 32 * w + __ffs(bits) - 1;
  V2 s, t;
  push_candidate(W.view(), S, C, c / C.na, c % C.na, false, s, t);
  if (l == 0) atomicAdd(reinterpret_cast<unsigned long long*>(&a.counters[3]), 1ull);
  double residual;
#ifdef PPG_PHASE_TRACE_BUILD
  PPG_PHASE_MARK(1, t_ph);
#endif
  const int st = warp_resolve_any<NW, kPoly>(W, G, O, S, C, pij, s, t, false, &residual);
#ifdef PPG_PHASE_TRACE_BUILD
  PPG_PHASE_MARK(2, t_ph);
#endif
  if (st != 0) {  // SimError: reward 0 (mcts.cpp:153-158)
    if (l == 0) {
      a.env_done[e] = 1;
      a.env_reward[e] = 0.0;
    }
    return 1;
  }
  const GraspOut gr = warp_graspable(W, S, C, a.S.target[0]);
#ifdef PPG_PHASE_TRACE_BUILD
  PPG_PHASE_MARK(3, t_ph);
#endif
  if (l == 0) {
    const int pushes = a.env_pushes[e] + 1;
    a.env_pushes[e] = pushes;
    if (gr.graspable) {
      a.env_done[e] = 1;
      a.env_bygrasp[e] = 1;
      a.env_reward[e] = C.gamma_pow[pushes];
    } else if (pushes >= a.cap) {
      a.env_done[e] = 1;
      a.env_reward[e] = 0.0;
    }
  }
  warp_store(W, env);
  return 1;
}

// RolloutCursor::step (mcts.cpp:142-171), one warp per active environment.
template <int NW, bool kPoly>
__global__ void __launch_bounds__(kWarpsPerBlock * 32) lock_step_warp_kernel(const __grid_constant__ SimConst C,
                                                                            LockArgs a) {
  PPG_POLY_SMEM
  lock_dyn(a);
  if (a.round_mode && *a.round_mode != 0) return;  // adaptive: a hybrid round
  __shared__ double blk[kWarpsPerBlock][160];
  __shared__ unsigned valid[kWarpsPerBlock][32];
  __shared__ uint16_t pij[kWarpMaxN * (kWarpMaxN - 1) / 2];
  build_pairs(pij, C.n);
  const int wib = threadIdx.x >> 5;
  const int gw = blockIdx.x * kWarpsPerBlock + wib;
  if (gw >= *a.n_active) return;
  const WarpPoly G{poly_wv[kPoly ? wib : 0], poly_cen[kPoly ? wib : 0]};
  warp_rollout_step<NW, kPoly>(C, a, a.active[gw], blk[wib], valid[wib], pij, G);
}

// ---------------------------------------------------------------------------
// Asynchronous lockstep (the latency-bound rounds of lockstep_simulate,
// pmbs.cpp:188-203): the reference's rounds are a barrier — every active env
// steps once, then the sequential harvest — so a round costs its SLOWEST
// env-step.  But an env's trajectory depends on the others only through the
// harvest of the round in which it finished by grasp (its re-purposing
// target, argmax of W at that round).  So envs run their steps back to back,
// each tagged with its round; a harvester warp performs the harvest of round
// r as soon as every env has finished round r, with W(r) accumulated by the
// steps of round r themselves (W[node] += cap - pushes of each env still
// running after its step), and an env finished by grasp waits only for the
// harvest of ITS round.  Every env sees exactly the steps, RNG draws and
// re-purposing decisions of the lockstep run, so results are bit-identical;
// the critical path becomes max over envs of their own chains instead of the
// sum over rounds of the slowest step.
//
// Ownership: env e is stepped only by worker warp (e mod n_workers), which
// is the only writer of its state (the harvester publishes a re-purposing
// decision in env_state and the owner applies it), so no env data crosses
// SMs except through the harvester's L2 reads of finished envs.  The ring of
// kAsyncK rounds bounds how far envs run ahead.  All warps must be resident
// (cooperative launch, grid <= occupancy); every wait is bounded by
// globaltimer (a stuck protocol sets the error word and exits).

PPG_DI int ld_volatile(const int32_t* p) { return *reinterpret_cast<const volatile int32_t*>(p); }
PPG_DI unsigned long long now_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
constexpr unsigned long long kAsyncStallNs = 20ull * 1000 * 1000 * 1000;  // 20 s without progress: error

// env_state values of the asynchronous / wave protocols
enum : int { kReady = 0, kAwait = 1, kGone = 2, kPhys = -1, kSpec = 4 };  // kSpec: a speculative step is held

// Ring views
PPG_DI int32_t* ring_ctr(const LockArgs& a, int r) { return a.a_ctr + kRingCtr * (r % kAsyncK); }
PPG_DI int32_t* ring_P(const LockArgs& a, int r) { return a.a_P + (r % kAsyncK) * a.a_wcap; }
PPG_DI int ld_acquire(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void lock_async_init_kernel(const __grid_constant__ SimConst C, LockArgs a) {
  lock_dyn(a);
  if (a.round_mode && *a.round_mode != 0) return;  // adaptive: a hybrid round
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int G = gridDim.x * blockDim.x;
  for (int e = tid; e < a.used; e += G) {
    a.env_round[e] = 0;
    a.env_state[e] = a.env_done[e] ? 2 : 0;  // the lockstep harvest just harvested every done env
    if (a.env_done[e]) atomicAdd(&a.a_ctl[2], 1);
  }
  for (int i = tid; i < kAsyncK * a.n_nodes; i += G) {
    a.a_W[(i / a.n_nodes) * a.a_wcap + i % a.n_nodes] = 0;
    a.a_P[(i / a.n_nodes) * a.a_wcap + i % a.n_nodes] = 0;
  }
  if (tid < kRingCtr * kAsyncK) a.a_ctr[tid] = 0;
}

#ifndef PPG_ASYNC_BLOCKS
#define PPG_ASYNC_BLOCKS 3  // resident blocks per SM the register budget is sized for
#endif
template <int NW, bool kPoly, bool kSpecul>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, PPG_ASYNC_BLOCKS) lock_async_kernel(const __grid_constant__ SimConst C,
                                                                           LockArgs a) {
  PPG_POLY_SMEM
  lock_dyn(a);
  int32_t* ctl = a.a_ctl;
  // runs in the asynchronous regime, or to finish a wave-round call once its
  // batch has shrunk (ctl[5] == 2: continues from the wave state)
  if (a.round_mode && *a.round_mode != 0 && ctl[5] != 2) return;
  __shared__ double blk[kWarpsPerBlock][160];
  __shared__ unsigned valid[kWarpsPerBlock][32];
  __shared__ uint16_t pij[kWarpMaxN * (kWarpMaxN - 1) / 2];
  build_pairs(pij, C.n);
  const int wib = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int gw = blockIdx.x * kWarpsPerBlock + wib;
  const int used = a.used;
  if (gw == 0) {
    // ---- harvester.  D = the last DECIDED round, F = the last COMPLETE round
    // (every env finished it or is gone); the re-purposing target of round
    // r (argmax W(r), pmbs.cpp:171-180) is decided as soon as it is robust to
    // the envs that have not finished round r yet: each of them can add at
    // most cap - 1 to one node's W (a not-done env contributes cap - pushes,
    // pushes >= 1), so max W_known > every other W_known + stragglers * (cap - 1)
    // fixes the argmax; with no straggler the decision is the exact one.
    int F = ld_volatile(&ctl[0]);
    int D = max(F, ld_volatile(&ctl[9]));  // rounds the wave harvests already decided
    const int F0 = F;              // round F0 + 1 is already counted (lock / wave setup)
    int G = ld_volatile(&ctl[2]);  // envs gone through round F
    unsigned long long t_idle = now_ns();
    {  // the workers' pending bounds of their READY envs are in place
      const int nwk = gridDim.x * kWarpsPerBlock - 1, owners = nwk < used ? nwk : used;
      while (ld_volatile(&ctl[10]) < owners) {
        if (now_ns() - t_idle > kAsyncStallNs) {
          if (l == 0) {
            atomicExch(&ctl[3], 1);
            atomicExch(&ctl[1], 1);
            if (a.cond) cudaGraphSetConditional(static_cast<cudaGraphConditionalHandle>(a.cond), 0u);
          }
          return;
        }
        __nanosleep(64);
      }
      __threadfence();
    }
    for (;;) {
      // finished when nothing will step in round F + 1.  Envs waiting on the
      // decision of round F add to gone(F + 1) only once they have applied it,
      // so this is re-checked every pass rather than only when F advances.
      if (G + ld_volatile(&ring_ctr(a, F + 1)[1]) >= used) {
        if (l == 0) {
          atomicExch(&ctl[1], 1);
          // the iteration graph's WHILE loop ends here (the wave path skips the lockstep harvest)
          if (a.cond) cudaGraphSetConditional(static_cast<cudaGraphConditionalHandle>(a.cond), 0u);
        }
        return;
      }
      bool progress = false;
      // decide round D + 1
      const int r = D + 1;
      if (r <= F + kAsyncK - 1) {
        int32_t* rc = ring_ctr(a, r);
        int gone_eff = G;
        for (int q = F + 1; q <= r; ++q) gone_eff += ld_volatile(&ring_ctr(a, q)[1]);
        const int arr = ld_acquire(&rc[0]);  // before near: a stale near may only over-count far
        const int strag = used - gone_eff - arr;
        if (strag > 0 || arr > 0) {
          // the envs that have not finished round r: those already READY for it
          // ("near", their node and bound cap - 1 - pushes in P(r)) and the
          // rest ("far": any node, at most cap - 1).  Read order: arrivals,
          // near / P (acquire), then W — a worker publishes W, then drops its
          // P bound, then counts its arrival, so every env is covered.
          const int near = ld_acquire(&rc[6]);
          const int far = strag - near;
          const int32_t* W = a.a_W + (r % kAsyncK) * a.a_wcap;
          const int32_t* Pr = ring_P(a, r);
          int m1 = 0, b1 = -1;
          for (int i = l; i < a.n_nodes; i += 32) {
            const int w = ld_volatile(&W[i]);
            if (w > m1) {
              m1 = w;
              b1 = i;
            }
          }
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) {
            const int om1 = __shfl_xor_sync(kFull, m1, off);
            const int ob1 = __shfl_xor_sync(kFull, b1, off);
            if (om1 > m1 || (om1 == m1 && om1 > 0 && ob1 < b1)) {
              m1 = om1;
              b1 = ob1;
            }
          }
          // the most any other node can still reach, split by its side of b1
          // (a tie goes to the lower node)
          int lo = 0, hi = 0, vb = 0, ib = -1;  // vb / ib: the likely outcome, argmax(W + P)
          for (int i = l; i < a.n_nodes; i += 32) {
            const int pi = ld_acquire(&Pr[i]);  // P before W
            const int v = pi + ld_volatile(&W[i]);
            if (i < b1) lo = max(lo, v);
            else if (i > b1) hi = max(hi, v);
            if (v > vb) {
              vb = v;
              ib = i;
            }
          }
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) {
            lo = max(lo, __shfl_xor_sync(kFull, lo, off));
            hi = max(hi, __shfl_xor_sync(kFull, hi, off));
            const int ov = __shfl_xor_sync(kFull, vb, off), oi = __shfl_xor_sync(kFull, ib, off);
            if (ov > vb || (ov == vb && ov > 0 && oi < ib)) {
              vb = ov;
              ib = oi;
            }
          }
          const int slack = far * (a.cap - 1);
          // (m1 from the first pass is a lower bound of W(r)[b1]; with m1 = 0,
          // hi covers every node with the fresher W of the second pass)
          const bool robust = strag == 0 || !a.leaf_parallel ||  // (no re-purposing: the decision is -1 anyway)
                              (a.n_nodes == 1 && m1 > 0) ||        // one node: nothing can overtake it
                              (far >= 0 && (m1 > 0 ? (lo + slack < m1 && hi + slack <= m1) : (far == 0 && hi == 0)));
          if (robust) {
            if (l == 0) {
              rc[4] = (a.leaf_parallel && m1 > 0) ? b1 : -1;
              __threadfence();
              atomicExch(&rc[3], r);  // decision of round r published
            }
            D = r;
            progress = true;
          } else if (kSpecul && l == 0 && a.leaf_parallel) {
            // not fixed yet: the likely decision, for speculative re-purposing
            const unsigned long long pv = static_cast<unsigned long long>(static_cast<unsigned>(r)) << 32 |
                                          static_cast<unsigned>(vb > 0 ? ib : -1);
            atomicExch(reinterpret_cast<unsigned long long*>(rc + 8), pv);
          }
        }
      }
      // advance F: round F + 1 is complete once every env has finished it or
      // is gone by then (envs that finished by grasp have applied the decision)
      {
        const int rf = F + 1;
        int32_t* rc = ring_ctr(a, rf);
        const int arrived = ld_volatile(&rc[0]);
        if (D >= rf && arrived == used - (G + ld_volatile(&rc[1]))) {
          G += ld_volatile(&rc[1]);
          // the lockstep harvest counts every round that runs
          if (l == 0 && rf > F0 + 1 && arrived > 0) a.counters[1] += 1;
          int32_t* Wm = a.a_W + (rf % kAsyncK) * a.a_wcap;
          for (int i = l; i < a.n_nodes; i += 32) Wm[i] = 0;
          __syncwarp();
          if (l == 0) {
            rc[0] = 0;
            rc[1] = 0;
            rc[2] = 0;
            __threadfence();
            atomicExch(&ctl[0], rf);  // round rf complete: its ring slot is free for round rf + K
          }
          F = rf;
          progress = true;
        }
      }
      if (progress) {
        t_idle = now_ns();
      } else {
        if (now_ns() - t_idle > kAsyncStallNs) {
          if (l == 0) {
            atomicExch(&ctl[3], 1);
            atomicExch(&ctl[1], 1);
            if (a.cond) cudaGraphSetConditional(static_cast<cudaGraphConditionalHandle>(a.cond), 0u);
          }
          return;
        }
        __nanosleep(64);
      }
    }
  }
  // ---- workers: warp w owns envs w, w + n_workers, ... (the only writer of their state)
  const int nwk = gridDim.x * kWarpsPerBlock - 1;
  const int wk = gw - 1;
  if (wk >= used) return;  // owns no env
  const WarpPoly G{poly_wv[kPoly ? wib : 0], poly_cen[kPoly ? wib : 0]};
  if (l == 0) {  // pending bounds of this warp's READY envs (fresh start or wave hand-over)
    for (int e = wk; e < used; e += nwk)
      if (a.env_state[e] == kReady) {
        const int r1 = a.env_round[e] + 1;
        atomicAdd(&ring_P(a, r1)[a.env_node[e]], a.cap - 1 - a.env_pushes[e]);
        atomicAdd(&ring_ctr(a, r1)[6], 1);
      }
    __threadfence();
    atomicAdd(&ctl[10], 1);
  }
  __syncwarp();
  unsigned long long t_idle = now_ns();
  for (;;) {
    int fin = 0, F = 0;
    if (l == 0) {
      fin = ld_volatile(&ctl[1]);
      F = ld_volatile(&ctl[0]);
    }
    fin = __shfl_sync(kFull, fin, 0);
    F = __shfl_sync(kFull, F, 0);
    if (fin) return;
    bool progress = false;
    for (int e = wk; e < used; e += nwk) {
      int st = l == 0 ? ld_volatile(&a.env_state[e]) : 0;
      st = __shfl_sync(kFull, st, 0);
      if (st == kAwait || st == kSpec) {
        // finished by grasp in round rho: apply the decision of rho once
        // published (pmbs.cpp:181-185); until then, step speculatively at the
        // likely decision and hold the result (kSpec): kept when the decision
        // agrees, discarded (cursor, RNG index and counters restored) when not
        int b = -2, spec_node = -1;
        if (l == 0) {
          const int rho = a.env_round[e];
          int32_t* rc = ring_ctr(a, rho);
          if (ld_volatile(&rc[3]) == rho) {
#ifdef PPG_PHASE_TRACE_BUILD
            {
              unsigned long long t_now;
              asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_now));
              atomicAdd(&g_phase_ns[5], t_now - g_await_t0[e & 65535]);
              atomicAdd(&g_phase_ns[6], 1ull);
            }
#endif
            __threadfence();
            b = ld_volatile(&rc[4]);
            bool kept = false;
            if (kSpecul && st == kSpec) {
              const int4 sp = a.a_spec[e];
              if (b == sp.x && a.mt_idx[e] < kMtFrozen) {  // the held step stands: publish it as round rho + 1
                kept = true;
                atomicAdd(reinterpret_cast<unsigned long long*>(&a.counters[2]), 1ull);
                const int r = rho + 1;
                int32_t* rc2 = ring_ctr(a, r);
                a.env_round[e] = r;
                const int node = a.env_node[e];
                if (!a.env_done[e]) atomicAdd(&a.a_W[(r % kAsyncK) * a.a_wcap + node], a.cap - a.env_pushes[e]);
                __threadfence();
                if (!a.env_done[e]) {
                  atomicAdd(&ring_P(a, r + 1)[node], a.cap - 1 - a.env_pushes[e]);
                  atomicAdd(&ring_ctr(a, r + 1)[6], 1);
                  a.env_state[e] = kReady;
                } else {
                  atomicMax(&a.rew[node], static_cast<unsigned long long>(__double_as_longlong(a.env_reward[e])));
                  a.env_harvested[e] = 1;
                  if (a.env_bygrasp[e]) {
                    a.env_state[e] = kAwait;
                  } else {
                    a.env_state[e] = kGone;
                    atomicAdd(&ring_ctr(a, r + 1)[1], 1);
                  }
                }
                __threadfence();
                atomicAdd(&rc2[0], 1);
                b = -3;  // handled
              } else {  // discard the held step: back to "finished by grasp, harvested"
                a.mt_idx[e] = sp.z;
                a.env_harvested[e] = 1;
                a.env_done[e] = 1;
                a.env_bygrasp[e] = 1;
                atomicAdd(reinterpret_cast<unsigned long long*>(&a.counters[0]), ~0ull);
                if (sp.w) atomicAdd(reinterpret_cast<unsigned long long*>(&a.counters[3]), ~0ull);
              }
            }
            if (!kept) {
              if (b >= 0) {  // re-purpose: RolloutCursor ctor at b, continues at round rho + 1
                cursor_init(C, a, e, b);
                a.env_harvested[e] = 0;
                atomicAdd(&ring_P(a, rho + 1)[b], a.cap - 1 - a.env_pushes[e]);
                atomicAdd(&ring_ctr(a, rho + 1)[6], 1);
                a.env_state[e] = kReady;
                atomicAdd(reinterpret_cast<unsigned long long*>(&a.counters[2]), 1ull);
              } else {
                a.env_state[e] = kGone;
                atomicAdd(&ring_ctr(a, rho + 1)[1], 1);  // does not step in round rho + 1
              }
            }
          } else if (kSpecul && st == kAwait && rho + 1 <= F + kAsyncK - 1 && a.mt_idx[e] < 312) {
            const unsigned long long pv = *reinterpret_cast<volatile unsigned long long*>(rc + 8);
            const int pn = static_cast<int>(static_cast<unsigned>(pv));
            if (static_cast<int>(pv >> 32) == rho && pn >= 0) spec_node = pn;
          }
        }
        b = __shfl_sync(kFull, b, 0);
        spec_node = __shfl_sync(kFull, spec_node, 0);
        __syncwarp();
        if (kSpecul && b == -2 && spec_node >= 0) {  // speculative step at the likely decision
          int p_before = 0, mt0 = 0;
          if (l == 0) {
            mt0 = a.mt_idx[e];
            cursor_init(C, a, e, spec_node);
            a.env_harvested[e] = 0;
            p_before = a.env_pushes[e];
          }
          __syncwarp();
          const int res = warp_rollout_step<NW, kPoly>(C, a, e, blk[wib], valid[wib], pij, G, true);
          __syncwarp();
          if (l == 0) {
            a.a_spec[e] = make_int4(spec_node, p_before, mt0, res);
            a.env_state[e] = kSpec;
          }
          __syncwarp();
          progress = true;
          continue;
        }
        if (b == -2) continue;
        progress = true;
        if (b == -3) continue;
        st = b >= 0 ? kReady : kGone;
      }
      if (st != kReady) continue;
      const int r = a.env_round[e] + 1;
      if (r > F + kAsyncK - 1) continue;  // ring bound: at most K rounds past the last complete round
      const int p_before = a.env_pushes[e];
      warp_rollout_step<NW, kPoly>(C, a, e, blk[wib], valid[wib], pij, G);
      __syncwarp();
      if (l == 0) {
        a.env_round[e] = r;
        int32_t* rc = ring_ctr(a, r);
        const int node = a.env_node[e];
        if (!a.env_done[e]) atomicAdd(&a.a_W[(r % kAsyncK) * a.a_wcap + node], a.cap - a.env_pushes[e]);
        __threadfence();  // W before the pending bound is dropped
        atomicSub(&ring_P(a, r)[node], a.cap - 1 - p_before);
        atomicSub(&rc[6], 1);
        if (!a.env_done[e]) {
          atomicAdd(&ring_P(a, r + 1)[node], a.cap - 1 - a.env_pushes[e]);
          atomicAdd(&ring_ctr(a, r + 1)[6], 1);
        } else {
          atomicMax(&a.rew[a.env_node[e]], static_cast<unsigned long long>(__double_as_longlong(a.env_reward[e])));
          a.env_harvested[e] = 1;
          if (a.leaf_parallel && a.env_bygrasp[e]) {
            a.env_state[e] = kAwait;  // waits for the decision of round r
#ifdef PPG_PHASE_TRACE_BUILD
            {
              unsigned long long t_now;
              asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_now));
              g_await_t0[e & 65535] = t_now;
            }
#endif
          } else {
            a.env_state[e] = kGone;
            atomicAdd(&ring_ctr(a, r + 1)[1], 1);  // does not step in round r + 1
          }
        }
        __threadfence();
        atomicAdd(&rc[0], 1);
      }
      __syncwarp();
      progress = true;
    }
    if (progress) {
      t_idle = now_ns();
    } else {
      if (now_ns() - t_idle > kAsyncStallNs) {
        if (l == 0) {
          atomicExch(&ctl[3], 2);
          atomicExch(&ctl[1], 1);
        }
        return;
      }
      __nanosleep(256);
    }
  }
}

// ---------------------------------------------------------------------------
// Wave rounds: the asynchronous lockstep for LARGE disc batches, where the
// physics must stay on the lane-per-env kernel (its throughput) and
// sample / graspable stay one warp per env.  Same protocol as
// lock_async_kernel (round-tagged steps, W(r) ring, in-order harvests), but
// driven by a loop of four ordinary launches ("waves") instead of one
// persistent kernel — no launch waits on another:
//   wave_harvest_kernel  harvests every complete round, then lists the envs
//                        that may start a step (READY, within the ring) and
//                        the yielded physics to resume;
//   wave_sample_kernel   sample + pick for the listed READY envs (one warp each);
//   resolve_disc_kernel<N, true> with a per-launch iteration budget: an env
//                        that exceeds it yields (progress saved) and resumes
//                        in the next wave, so one jammed push no longer holds
//                        up the 64K envs of a barrier round;
//   wave_post_kernel     graspable + reward + the round's bookkeeping.
// Env states: 0 READY, 1 AWAIT (finished by grasp, awaits the harvest of
// its round), 2 GONE, -1 PHYS (physics pending / yielded).


// The end of env e's step of round r (lane 0): W(r) for an env still running,
// else the round's done list; arrival last (after a fence).
PPG_DI void wave_step_done(const LockArgs& a, int e, int r) {
  int32_t* rc = ring_ctr(a, r);
  if (!a.env_done[e]) {
    atomicAdd(&a.a_W[(r % kAsyncK) * a.a_wcap + a.env_node[e]], a.cap - a.env_pushes[e]);
    a.env_state[e] = kReady;
  } else {
    // the reward max is order-free: folded in as the env finishes (the
    // asynchronous kernel continuing a wave-round call relies on it)
    atomicMax(&a.rew[a.env_node[e]], static_cast<unsigned long long>(__double_as_longlong(a.env_reward[e])));
    a.env_harvested[e] = 1;
    a.a_dl[static_cast<size_t>(r % kAsyncK) * a.E + atomicAdd(&rc[2], 1)] = e;
    if (a.leaf_parallel && a.env_bygrasp[e]) {
      a.env_state[e] = kAwait;
    } else {
      a.env_state[e] = kGone;
      atomicAdd(&ring_ctr(a, r + 1)[1], 1);
    }
  }
  a.env_round[e] = r;
  __threadfence();
  atomicAdd(&rc[0], 1);
}

// (max, first index of the max, largest other value) merge of two partial
// scans of W (strict >, W > 0, lowest node wins a tie: pmbs.cpp:171-180)
PPG_DI void top2_merge(int& m1, int& b1, int& m2, int om1, int ob1, int om2) {
  if (om1 > m1 || (om1 == m1 && om1 > 0 && ob1 < b1)) {
    m2 = max(m2, max(m1, om2));
    m1 = om1;
    b1 = ob1;
  } else {
    m2 = max(m2, max(om1, om2));
  }
}

// Sharded wave rounds: this shard's W ring and per-slot (arrived, gone)
// counts into g_ring, which the host then all-reduces (sum) over the shards.
// Before the call's first wave (nothing initialised yet) the contribution is 0.
__global__ void wave_pack_kernel(LockArgs a) {
  lock_dyn(a);
  const int P = a.n_nodes;
  const bool fresh = a.a_ctl[4] == 0;
  // [K][P] W | [K][2] (arrived, gone) | round r_p | near | P(r_p)[P]: the
  // pending bounds of the envs READY for the next undecided round r_p
  // (r_p from shard 0 only, so the sum is r_p; wave_pack_pending_kernel
  // adds the bounds)
  const int total = kAsyncK * P + 2 * kAsyncK + 2 + P;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    int v = 0;
    if (!fresh) {
      if (i < kAsyncK * P) {
        v = a.a_W[(i / P) * a.a_wcap + i % P];
      } else if (i < kAsyncK * P + 2 * kAsyncK) {
        const int k = i - kAsyncK * P;
        v = a.a_ctr[kRingCtr * (k >> 1) + (k & 1)];
      } else if (i == kAsyncK * P + 2 * kAsyncK && a.shard_r == 0) {
        v = a.a_ctl[9] + 1;
      }
    }
    a.g_ring[i] = v;
  }
}

__global__ void wave_pack_pending_kernel(LockArgs a) {
  lock_dyn(a);
  if (a.a_ctl[4] == 0) return;
  const int P = a.n_nodes;
  const int rp = a.a_ctl[9] + 1;
  int32_t* near = a.g_ring + kAsyncK * P + 2 * kAsyncK + 1;
  int32_t* Pp = near + 1;
  int cnt = 0;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < a.used; e += gridDim.x * blockDim.x) {
    const int st = a.env_state[e];
    if ((st == kReady || st == kPhys) && a.env_round[e] + 1 == rp) {
      atomicAdd(&Pp[a.env_node[e]], a.cap - 1 - a.env_pushes[e]);
      ++cnt;
    }
  }
  if (cnt) atomicAdd(near, cnt);
}

// Between waves (one block): decide every round whose re-purposing target is
// already fixed (the early decision of lock_async_kernel: max W_known > every
// other W_known + stragglers * (cap - 1)), apply the decisions to the
// by-grasp envs waiting on them, complete rounds in order, then the wave's
// lists.  a_ctl: [0] complete round F, [2] envs gone through round F,
// [4] set up, [9] decided round D.  Ring slot: [0] arrived, [1] gone at this
// round, [2] done-list length, [3] decided round, [4] decision, [5] done-list
// entries already applied.
__global__ void __launch_bounds__(1024) wave_harvest_kernel(const __grid_constant__ SimConst C, LockArgs a) {
  lock_dyn(a);
  if (a.round_mode && *a.round_mode == 0) return;  // this lockstep call runs asynchronously
  const int tid = threadIdx.x, B = blockDim.x, lane = tid & 31, wid = tid >> 5;
  const int used = a.used;
  int32_t* ctl = a.a_ctl;
  // decisions, completion and termination read the batch-wide values: this
  // context's own ring, or (sharded) the ring summed over the shards
  const bool sharded = a.g_ring != nullptr;
  const int used_g = sharded ? a.used_global : used;
  const int P = a.n_nodes;
  auto W_of = [&](int r) -> const int32_t* {
    return sharded ? a.g_ring + (r % kAsyncK) * P : a.a_W + (r % kAsyncK) * a.a_wcap;
  };
  auto arr_of = [&](int r) { return sharded ? a.g_ring[kAsyncK * P + 2 * (r % kAsyncK)] : ring_ctr(a, r)[0]; };
  auto gone_of = [&](int r) { return sharded ? a.g_ring[kAsyncK * P + 2 * (r % kAsyncK) + 1] : ring_ctr(a, r)[1]; };
  __shared__ int s_H, s_G, s_D, s_ns, s_np, s_prog, s_strag, s_try, s_F0, s_near, s_usep;
  __shared__ int s_m1[32], s_b1[32], s_m2[32], s_rep[32], s_ret[32], s_lo[32], s_hi[32];
  constexpr int kWaveP = 4096;  // pending bounds kept per node in shared memory up to this many nodes
  __shared__ int s_P[kWaveP];
  if (ctl[4] == 0) {  // first wave of the call: every env READY or GONE at round 0
    if (tid == 0) s_G = 0;
    __syncthreads();
    int g = 0;
    for (int e = tid; e < used; e += B) {
      a.env_round[e] = 0;
      a.env_state[e] = a.env_done[e] ? kGone : kReady;
      a.resume_si[e] = -1;
      g += a.env_done[e] ? 1 : 0;
    }
    for (int i = tid; i < kAsyncK * a.n_nodes; i += B) {
      a.a_W[(i / a.n_nodes) * a.a_wcap + i % a.n_nodes] = 0;
      a.a_P[(i / a.n_nodes) * a.a_wcap + i % a.n_nodes] = 0;  // the asynchronous hand-over rebuilds it
    }
    if (tid < kRingCtr * kAsyncK) a.a_ctr[tid] = 0;
    atomicAdd(&s_G, g);
    __syncthreads();
    if (tid == 0) {
      ctl[0] = 0;
      if (sharded) {  // the batch-wide count arrives with the next exchange: gone at round 1
        ring_ctr(a, 1)[1] = s_G;
        ctl[2] = 0;
      } else {
        ctl[2] = s_G;
      }
      ctl[4] = 1;
      ctl[9] = 0;
    }
    __syncthreads();
  }
  if (tid == 0) {
    s_H = ctl[0];
    s_G = ctl[2];
    s_D = ctl[9];
    s_F0 = s_H;
  }
  __syncthreads();
  for (;;) {
    __syncthreads();  // every thread has read the previous pass's shared state
    if (tid == 0) {
      s_prog = 0;
      // (1) can round D + 1 be decided?
      const int r = s_D + 1;
      s_try = 0;
      // sharded: only rounds whose slot the exchange of this wave carried
      // (a slot freed in this pass still holds its old round's sums)
      if (r <= s_H + kAsyncK - 1 && (!sharded || r <= s_F0 + kAsyncK - 1)) {
        int gone_eff = s_G;
        for (int q = s_H + 1; q <= r; ++q) gone_eff += gone_of(q);
        const int arr = arr_of(r);
        s_strag = used_g - gone_eff - arr;
        s_try = (s_strag > 0 || arr > 0) ? 1 : 0;
      }
    }
    __syncthreads();
    if (s_try) {
      const int r = s_D + 1;
      const int32_t* W = W_of(r);
      // pending bounds of the envs READY (or in physics) for round r: their
      // node and cap - 1 - pushes (lock_async_kernel's rule); sharded, the
      // summed bounds of the exchange when they are for this round
      const int32_t* gP = nullptr;
      if (tid == 0) {
        s_usep = 0;
        s_near = 0;
        if (sharded) {
          const int base = kAsyncK * P + 2 * kAsyncK;
          if (a.g_ring[base] == r) {
            s_usep = 2;
            s_near = a.g_ring[base + 1];
          }
        } else if (a.leaf_parallel && a.n_nodes > 1 && a.n_nodes <= kWaveP) {
          s_usep = 1;  // (one node: no competitor, decided below without the scan)
        }
      }
      __syncthreads();
      if (s_usep == 1) {
        for (int i = tid; i < a.n_nodes; i += B) s_P[i] = 0;
        __syncthreads();
        int cnt = 0;
        for (int e = tid; e < used; e += B) {
          const int st = a.env_state[e];
          if ((st == kReady || st == kPhys) && a.env_round[e] + 1 == r) {
            atomicAdd(&s_P[a.env_node[e]], a.cap - 1 - a.env_pushes[e]);
            ++cnt;
          }
        }
        if (cnt) atomicAdd(&s_near, cnt);
        __syncthreads();
      } else if (s_usep == 2) {
        gP = a.g_ring + kAsyncK * P + 2 * kAsyncK + 2;
      }
      int m1 = 0, b1 = -1, m2 = 0;
      for (int i = tid; i < a.n_nodes; i += B) top2_merge(m1, b1, m2, W[i], i, 0);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1)
        top2_merge(m1, b1, m2, __shfl_xor_sync(kFull, m1, off), __shfl_xor_sync(kFull, b1, off),
                   __shfl_xor_sync(kFull, m2, off));
      if (lane == 0) {
        s_m1[wid] = m1;
        s_b1[wid] = b1;
        s_m2[wid] = m2;
      }
      __syncthreads();
      if (tid < 32) {
        const int nw = B >> 5;
        m1 = tid < nw ? s_m1[tid] : 0;
        b1 = tid < nw ? s_b1[tid] : -1;
        m2 = tid < nw ? s_m2[tid] : 0;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1)
          top2_merge(m1, b1, m2, __shfl_xor_sync(kFull, m1, off), __shfl_xor_sync(kFull, b1, off),
                     __shfl_xor_sync(kFull, m2, off));
        if (tid == 0) {
          s_m1[0] = m1;  // broadcast (m1, b1, m2) for the pending-bound pass
          s_b1[0] = b1;
          s_m2[0] = m2;
        }
      }
      __syncthreads();
      m1 = s_m1[0];
      b1 = s_b1[0];
      m2 = s_m2[0];
      __syncthreads();
      int lo = 0, hi = 0;
      if (s_usep) {  // the most any other node can still reach, by its side of b1
        for (int i = tid; i < a.n_nodes; i += B) {
          const int v = W[i] + (s_usep == 1 ? s_P[i] : gP[i]);
          if (i < b1) lo = max(lo, v);
          else if (i > b1) hi = max(hi, v);
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          lo = max(lo, __shfl_xor_sync(kFull, lo, off));
          hi = max(hi, __shfl_xor_sync(kFull, hi, off));
        }
        if (lane == 0) {
          s_lo[wid] = lo;
          s_hi[wid] = hi;
        }
        __syncthreads();
        if (tid == 0) {
          for (int w = 1; w < (B >> 5); ++w) {
            lo = max(lo, s_lo[w]);
            hi = max(hi, s_hi[w]);
          }
        }
      }
      if (tid == 0) {
        const int strag = s_strag;
        bool robust = strag == 0 || !a.leaf_parallel ||  // (no re-purposing: the decision is -1 anyway)
                      (a.n_nodes == 1 && m1 > 0);          // one node: nothing can overtake it
        if (!robust && s_usep) {
          const int far = strag - s_near, slack = far * (a.cap - 1);
          robust = far >= 0 && (m1 > 0 ? (lo + slack < m1 && hi + slack <= m1) : (far == 0 && hi == 0));
        }
        if (!robust) robust = m1 > 0 && m2 + strag * (a.cap - 1) < m1;
        if (robust) {
          int32_t* rc = ring_ctr(a, r);
          rc[4] = (a.leaf_parallel && m1 > 0) ? b1 : -1;
          rc[3] = r;
          s_D = r;
          s_prog = 1;
        }
      }
      __syncthreads();
    }
    // (2) apply the decided rounds' decisions to their newly listed done envs
    for (int q = s_H + 1; q <= s_D; ++q) {
      int32_t* rc = ring_ctr(a, q);
      const int k0 = rc[5], nd = rc[2];
      if (k0 == nd) continue;
      const int best = rc[4];
      const int32_t* dl = a.a_dl + static_cast<size_t>(q % kAsyncK) * a.E;
      int rep = 0, ret = 0;
      for (int k = k0 + tid; k < nd; k += B) {
        const int e = dl[k];
        if (a.env_state[e] == kAwait) {
          if (best >= 0) {  // re-purpose (pmbs.cpp:181-185): a new cursor at best, continues at round q + 1
            cursor_init(C, a, e, best);
            a.env_harvested[e] = 0;
            a.env_state[e] = kReady;
            ++rep;
          } else {
            a.env_state[e] = kGone;
            ++ret;
          }
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        rep += __shfl_xor_sync(kFull, rep, off);
        ret += __shfl_xor_sync(kFull, ret, off);
      }
      if (lane == 0) {
        s_rep[wid] = rep;
        s_ret[wid] = ret;
      }
      __syncthreads();
      if (tid == 0) {
        int tr = 0, tt = 0;
        for (int w = 0; w < (B >> 5); ++w) {
          tr += s_rep[w];
          tt += s_ret[w];
        }
        a.counters[2] += tr;
        ring_ctr(a, q + 1)[1] += tt;  // retired: do not step in round q + 1
        rc[5] = nd;
      }
      __syncthreads();
    }
    // (3) complete round F + 1: decided, every env finished it or is gone, its done list applied
    const int r = s_H + 1;
    int32_t* rc = ring_ctr(a, r);
    const int gone_r = s_G + gone_of(r);
    if (gone_r >= used_g || s_D < r || arr_of(r) < used_g - gone_r) {
      if (!s_prog) break;
      continue;
    }
    int32_t* Wm = a.a_W + (r % kAsyncK) * a.a_wcap;
    for (int i = tid; i < a.n_nodes; i += B) Wm[i] = 0;
    __syncthreads();
    if (tid == 0) {
      rc[0] = 0;
      rc[1] = 0;
      rc[2] = 0;
      rc[5] = 0;
      s_G = gone_r;
      s_H = r;
      // the lockstep harvest counts every round that runs.  Sharded, gone(r + 1)
      // may still miss this pass's retirements, so round r itself is counted
      // (round 1 by the initial harvest)
      if (sharded ? (r >= 2 && arr_of(r) > 0) : (s_G + gone_of(r + 1) < used_g)) a.counters[1] += 1;
    }
    __syncthreads();
  }
  // lists of this wave: READY envs within the ring, yielded physics
  if (tid == 0) {
    s_ns = 0;
    s_np = 0;
    *a.n_stepping = 0;
    *a.fin_count = 0;
  }
  __syncthreads();
  const int H = s_H;
  for (int e0 = 0; e0 < used; e0 += B) {
    const int e = e0 + tid;
    const int st = e < used ? a.env_state[e] : kGone;
    const bool smp = st == kReady && a.env_round[e] + 1 <= H + kAsyncK - 1;
    const bool phy = st == kPhys;
    const unsigned ms = __ballot_sync(kFull, smp), mp = __ballot_sync(kFull, phy);
    int bs = 0, bp = 0;
    if (lane == 0) {
      if (ms) bs = atomicAdd(&s_ns, __popc(ms));
      if (mp) bp = atomicAdd(&s_np, __popc(mp));
    }
    bs = __shfl_sync(kFull, bs, 0);
    bp = __shfl_sync(kFull, bp, 0);
    const unsigned below = (1u << lane) - 1u;
    if (smp) a.active[bs + __popc(ms & below)] = e;
    if (phy) a.stepping[bp + __popc(mp & below)] = e;
  }
  __syncthreads();
  if (tid == 0) {
    ctl[0] = s_H;
    ctl[2] = s_G;
    ctl[9] = s_D;
    *a.n_active = s_ns;
    *a.n_stepping = s_np;
    const bool finished = s_G + gone_of(s_H + 1) >= used_g;
    // a shrunken batch: finish the yielded pushes unbounded in this wave
    // (no new samples), then the asynchronous kernel continues the rounds
    // (switch on the envs still running, not on the in-flight count: envs
    // held back by the ring bound are still work for the batch)
    const int remaining = used_g - (s_G + gone_of(s_H + 1));
    if (!finished && remaining < a.wave_switch) {
      ctl[5] = 2;
      ctl[8] = 0x7fffffff;
      *a.n_active = 0;
    } else {
      ctl[8] = a.wave_budget;
    }
    bool go = !finished;
    if (a.round_guard && go && ++*a.round_guard > kLockRoundLimit) {
      *a.round_guard = -1;  // a non-terminating protocol: reported by the host
      go = false;
    }
    if (a.go) *a.go = go ? 1 : 0;
    if (a.cond) cudaGraphSetConditional(static_cast<cudaGraphConditionalHandle>(a.cond), go ? 1u : 0u);
  }
}

// Sample + pick (mcts.cpp:145-152) for the wave's READY envs; a push goes to
// the physics list (fresh progress), no legal push ends the step (reward 0).
__global__ void __launch_bounds__(kWarpsPerBlock * 32) wave_sample_kernel(const __grid_constant__ SimConst C,
                                                                         LockArgs a) {
  lock_dyn(a);
  if (a.round_mode && *a.round_mode == 0) return;
  __shared__ double blk[kWarpsPerBlock][160];
  __shared__ unsigned valid[kWarpsPerBlock][32];
  const int wib = threadIdx.x >> 5;
  const int gw = blockIdx.x * kWarpsPerBlock + wib;
  if (gw >= *a.n_active) return;
  const int e = a.active[gw];
  const int n = C.n, l = threadIdx.x & 31;
  WarpEnv W(blk[wib], n, l);
  const ShapeView S = a.S.view(0);
  warp_load(W, a.env_poses + static_cast<size_t>(e) * n * 3, S);
  if (l == 0) atomicAdd(reinterpret_cast<unsigned long long*>(&a.counters[0]), 1ull);
  const int count = warp_sample_mask(W, S, C, valid[wib]);
  if (count == 0) {  // no legal push: reward 0 (mcts.cpp:146-150)
    if (l == 0) {
      a.env_done[e] = 1;
      a.env_reward[e] = 0.0;
      wave_step_done(a, e, a.env_round[e] + 1);
    }
    return;
  }
  const MtView g{a.mt + e, a.E};
  int idx = a.mt_idx[e];
  const uint64_t k = warp_mt_pick(g, idx, static_cast<uint64_t>(count), l);
  if (l == 0) a.mt_idx[e] = idx;
  int w = 0, seen = 0;
  while (seen + __popc(valid[wib][w]) <= static_cast<int>(k)) seen += __popc(valid[wib][w++]);
  unsigned bits = valid[wib][w];
  for (int drop = static_cast<int>(k) - seen; drop > 0; --drop) bits &= bits - 1;
  const int c = 32 * w + __ffs(bits) - 1;
  if (l == 0) {
    V2 s, t;
    push_candidate(W.view(), S, C, c / C.na, c % C.na, false, s, t);
    double* pu = a.env_push + static_cast<size_t>(e) * 4;
    pu[0] = s.x;
    pu[1] = s.y;
    pu[2] = t.x;
    pu[3] = t.y;
    a.resume_si[e] = -1;
    a.env_state[e] = kPhys;
    a.stepping[atomicAdd(a.n_stepping, 1)] = e;
  }
}

// The rest of RolloutCursor::step (mcts.cpp:153-170) for the envs whose
// physics finished in this wave, and the round's bookkeeping.
__global__ void __launch_bounds__(kWarpsPerBlock * 32) wave_post_kernel(const __grid_constant__ SimConst C,
                                                                       LockArgs a) {
  lock_dyn(a);
  if (a.round_mode && *a.round_mode == 0) return;
  __shared__ double blk[kWarpsPerBlock][160];
  const int wib = threadIdx.x >> 5;
  const int gw = blockIdx.x * kWarpsPerBlock + wib;
  if (gw >= *a.fin_count) return;
  const int e = a.fin_list[gw];
  const int n = C.n, l = threadIdx.x & 31;
  if (l == 0) atomicAdd(reinterpret_cast<unsigned long long*>(&a.counters[3]), 1ull);
  if (a.env_status[e] != 0) {  // SimError (mcts.cpp:153-158)
    if (l == 0) {
      a.env_done[e] = 1;
      a.env_reward[e] = 0.0;
      wave_step_done(a, e, a.env_round[e] + 1);
    }
    return;
  }
  WarpEnv W(blk[wib], n, l);
  const ShapeView S = a.S.view(0);
  warp_load(W, a.env_poses + static_cast<size_t>(e) * n * 3, S);
  const GraspOut gr = warp_graspable(W, S, C, a.S.target[0]);
  if (l == 0) {
    const int pushes = a.env_pushes[e] + 1;
    a.env_pushes[e] = pushes;
    if (gr.graspable) {
      a.env_done[e] = 1;
      a.env_bygrasp[e] = 1;
      a.env_reward[e] = C.gamma_pow[pushes];
    } else if (pushes >= a.cap) {
      a.env_done[e] = 1;
      a.env_reward[e] = 0.0;
    }
    wave_step_done(a, e, a.env_round[e] + 1);
  }
}

// Hybrid lockstep round for large disc batches: the sampler + pick and the
// graspable check of RolloutCursor::step (mcts.cpp:142-171) one warp per env
// (their candidate / angle loops spread over the lanes), the physics in
// between on the lane-per-env disc kernel (resolve_disc.cu, in place through
// the `stepping` list).  Phase 1: sample + pick.
__global__ void __launch_bounds__(kWarpsPerBlock * 32) lock_sample_warp_kernel(const __grid_constant__ SimConst C,
                                                                              LockArgs a) {
  lock_dyn(a);
  if (a.round_mode && *a.round_mode == 0) return;  // adaptive: a one-warp-per-env round
  __shared__ double blk[kWarpsPerBlock][160];
  __shared__ unsigned valid[kWarpsPerBlock][32];
  const int wib = threadIdx.x >> 5;
  const int gw = blockIdx.x * kWarpsPerBlock + wib;
  if (gw >= *a.n_active) return;
  const int e = a.active[gw];
  const int n = C.n, l = threadIdx.x & 31;
  WarpEnv W(blk[wib], n, l);
  const ShapeView S = a.S.view(0);
  warp_load(W, a.env_poses + static_cast<size_t>(e) * n * 3, S);
  if (l == 0) atomicAdd(reinterpret_cast<unsigned long long*>(&a.counters[0]), 1ull);
  const int count = warp_sample_mask(W, S, C, valid[wib]);
  if (count == 0) {  // no legal push: reward 0 (mcts.cpp:146-150)
    if (l == 0) {
      a.env_done[e] = 1;
      a.env_reward[e] = 0.0;
    }
    return;
  }
  const MtView g{a.mt + e, a.E};
  int idx = a.mt_idx[e];
  const uint64_t k = warp_mt_pick(g, idx, static_cast<uint64_t>(count), l);
  if (l == 0) a.mt_idx[e] = idx;
  int w = 0, seen = 0;
  while (seen + __popc(valid[wib][w]) <= static_cast<int>(k)) seen += __popc(valid[wib][w++]);
  unsigned bits = valid[wib][w];
  for (int drop = static_cast<int>(k) - seen; drop > 0; --drop) bits &= bits - 1;
  const int c = 32 * w + __ffs(bits) - 1;
  if (l == 0) {
    V2 s, t;
    push_candidate(W.view(), S, C, c / C.na, c % C.na, false, s, t);
    double* pu = a.env_push + static_cast<size_t>(e) * 4;
    pu[0] = s.x;
    pu[1] = s.y;
    pu[2] = t.x;
    pu[3] = t.y;
    a.stepping[atomicAdd(a.n_stepping, 1)] = e;
  }
}

// Phase 3: the rest of RolloutCursor::step for the envs the physics kernel
// resolved (SimError -> reward 0; else count the push, graspable, reward).
__global__ void __launch_bounds__(kWarpsPerBlock * 32) lock_post_warp_kernel(const __grid_constant__ SimConst C,
                                                                            LockArgs a) {
  lock_dyn(a);
  if (a.round_mode && *a.round_mode == 0) return;  // adaptive: a one-warp-per-env round
  __shared__ double blk[kWarpsPerBlock][160];
  const int wib = threadIdx.x >> 5;
  const int gw = blockIdx.x * kWarpsPerBlock + wib;
  const int n_st = *a.n_stepping;
  if (gw == 0 && (threadIdx.x & 31) == 0)
    atomicAdd(reinterpret_cast<unsigned long long*>(&a.counters[3]), static_cast<unsigned long long>(n_st));
  if (gw >= n_st) return;
  const int e = a.stepping[gw];
  const int n = C.n, l = threadIdx.x & 31;
  if (a.env_status[e] != 0) {  // SimError (mcts.cpp:153-158)
    if (l == 0) {
      a.env_done[e] = 1;
      a.env_reward[e] = 0.0;
    }
    return;
  }
  WarpEnv W(blk[wib], n, l);
  const ShapeView S = a.S.view(0);
  warp_load(W, a.env_poses + static_cast<size_t>(e) * n * 3, S);
  const GraspOut gr = warp_graspable(W, S, C, a.S.target[0]);
  if (l == 0) {
    const int pushes = a.env_pushes[e] + 1;
    a.env_pushes[e] = pushes;
    if (gr.graspable) {
      a.env_done[e] = 1;
      a.env_bygrasp[e] = 1;
      a.env_reward[e] = C.gamma_pow[pushes];
    } else if (pushes >= a.cap) {
      a.env_done[e] = 1;
      a.env_reward[e] = 0.0;
    }
  }
}

#define PPG_WARP_INST(NW, P)                                                                            \
  template __global__ void resolve_warp_kernel<NW, P>(const __grid_constant__ SimConst, ResolveArgs);  \
  template __global__ void expand_warp_kernel<NW, P>(const __grid_constant__ SimConst, ExpandArgs);    \
  template __global__ void lock_step_warp_kernel<NW, P>(const __grid_constant__ SimConst, LockArgs);        \
  template __global__ void lock_async_kernel<NW, P, false>(const __grid_constant__ SimConst, LockArgs); \
  template __global__ void lock_async_kernel<NW, P, true>(const __grid_constant__ SimConst, LockArgs);
PPG_WARP_INST(1, false)
PPG_WARP_INST(2, false)
PPG_WARP_INST(4, false)
PPG_WARP_INST(8, false)
PPG_WARP_INST(1, true)
PPG_WARP_INST(2, true)
PPG_WARP_INST(4, true)
#undef PPG_WARP_INST

}  // namespace ppg

// Latency split of the asynchronous kernel's env-steps (experiments): copies
// the PPG_PHASE_TRACE_BUILD accumulators to out[8] and zeroes them; returns
// PPG_EINVAL when the library was built without them.
extern "C" int ppg_debug_phase_times(unsigned long long* out) {
#ifdef PPG_PHASE_TRACE_BUILD
  if (cudaMemcpyFromSymbol(out, ppg::g_phase_ns, sizeof(unsigned long long) * 8) != cudaSuccess) return PPG_ECUDA;
  const unsigned long long zero[8] = {};
  if (cudaMemcpyToSymbol(ppg::g_phase_ns, zero, sizeof zero) != cudaSuccess) return PPG_ECUDA;
  return PPG_SUCCESS;
#else
  (void)out;
  return PPG_EINVAL;
#endif
}
