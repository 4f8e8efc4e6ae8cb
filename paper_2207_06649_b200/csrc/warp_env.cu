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

namespace ppg {

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
  const int e = a.active[gw];
  const int n = C.n, l = threadIdx.x & 31;
  WarpEnv W(blk[wib], n, l);
  const ShapeView S = a.S.view(0);
  double* env = a.env_poses + static_cast<size_t>(e) * n * 3;
  const WarpPoly G{poly_wv[kPoly ? wib : 0], poly_cen[kPoly ? wib : 0]};
  const PolyShape O = warp_load_any<kPoly>(W, G, env, S);
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
  // k-th valid candidate in (object, angle) order
  int w = 0, seen = 0;
  while (seen + __popc(valid[wib][w]) <= static_cast<int>(k)) seen += __popc(valid[wib][w++]);
  unsigned bits = valid[wib][w];
  for (int drop = static_cast<int>(k) - seen; drop > 0; --drop) bits &= bits - 1;
  const int c = 32 * w + __ffs(bits) - 1;
  V2 s, t;
  push_candidate(W.view(), S, C, c / C.na, c % C.na, false, s, t);
  if (l == 0) atomicAdd(reinterpret_cast<unsigned long long*>(&a.counters[3]), 1ull);
  double residual;
  const int st = warp_resolve_any<NW, kPoly>(W, G, O, S, C, pij, s, t, false, &residual);
  if (st != 0) {  // SimError: reward 0 (mcts.cpp:153-158)
    if (l == 0) {
      a.env_done[e] = 1;
      a.env_reward[e] = 0.0;
    }
    return;
  }
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
  warp_store(W, env);
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
  template __global__ void lock_step_warp_kernel<NW, P>(const __grid_constant__ SimConst, LockArgs);
PPG_WARP_INST(1, false)
PPG_WARP_INST(2, false)
PPG_WARP_INST(4, false)
PPG_WARP_INST(8, false)
PPG_WARP_INST(1, true)
PPG_WARP_INST(2, true)
PPG_WARP_INST(4, true)
#undef PPG_WARP_INST

}  // namespace ppg
