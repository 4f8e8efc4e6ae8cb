// warp_env.cu — latency mode: ONE WARP PER ENVIRONMENT (disc scenes, n <= 23).
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

#include "kernels.cuh"

namespace ppg {

constexpr int kWarpMaxN = 23;   // pair masks: 8 ballot words (253 pairs)
constexpr int kWarpWords = 8;
constexpr int kWarpsPerBlock = 4;

namespace {

constexpr unsigned kFull = 0xffffffffu;

// Per-warp shared block: x[n] | y[n] | theta[n] | cos | sin contiguous (a
// stride-1 PoseView, so the lane-level physics.cuh helpers apply), radii at
// [128, 160).  Latency mode runs disc scenes only, so the trig planes stay
// unused.
struct WarpEnv {
  double* x;
  double* y;
  double* th;
  double* r;
  int n;
  int lane;
  PPG_DI WarpEnv(double* blk, int n_, int lane_) : x(blk), y(blk + n_), th(blk + 2 * n_), r(blk + 128), n(n_), lane(lane_) {}
  PPG_DI PoseView view() const { return PoseView{x, 1, n}; }
};

PPG_DI double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = dmax(v, __shfl_xor_sync(kFull, v, o));
  return v;
}

// Builds the block's pair table for n objects: pij[p] = i | j << 8 (lexicographic).
PPG_DI void build_pairs(uint16_t* pij, int n) {
  if (threadIdx.x == 0) {
    int p = 0;
    for (int i = 0; i < n; ++i)
      for (int j = i + 1; j < n; ++j, ++p) pij[p] = static_cast<uint16_t>(i | (j << 8));
  }
  __syncthreads();
}

// Loads environment poses ([n][3] AoS) and radii into the warp's block.
PPG_DI void warp_load(WarpEnv& W, const double* poses, const ShapeView& S) {
  const int l = W.lane;
  if (l < W.n) {
    W.x[l] = poses[l * 3];
    W.y[l] = poses[l * 3 + 1];
    W.th[l] = poses[l * 3 + 2];
    W.r[l] = S.rad_(l);
  }
  __syncwarp();
}

PPG_DI void warp_store(const WarpEnv& W, double* poses) {
  const int l = W.lane;
  if (l < W.n) {
    poses[l * 3] = W.x[l];
    poses[l * 3 + 1] = W.y[l];
    poses[l * 3 + 2] = W.th[l];
  }
  __syncwarp();
}

// resolve_push (push_sim.cpp:58-130) for a disc scene, one warp.  Returns
// 0 ok, 1 start collision, 2 not converged (uniform); *residual = final max
// pairwise penetration.
//
// Register-centric: lane l OWNS object l (x, y, r in registers); every lane
// keeps register copies of the positions of its pairs (p = 32w + l) and their
// squared reach, refreshed by shuffles from the owners after the tip phase
// and patched in place after each pair hit (the moved positions are
// warp-uniform values).  No shared memory and no __syncwarp inside the
// iteration: shuffles and ballots are the only cross-lane traffic.  The
// block's shared pose copy is written back at the end for the sampler /
// grasp helpers.
PPG_DI int warp_resolve(WarpEnv& W, const SimConst& C, const uint16_t* pij, V2 start, V2 end, bool check_start,
                        double* residual) {
  const int n = W.n, l = W.lane;
  __syncwarp();
  const bool real = l < n;
  double xo = real ? W.x[l] : 0.0, yo = real ? W.y[l] : 0.0;
  const double ro = real ? W.r[l] : 0.0;
  if (check_start) {  // collides_gripper_start (world.cpp:154-164)
    const double rr = C.tip_r + C.tip_clear;
    const double h = C.side / 2.0;
    const bool wall = start.x - rr < -h || start.x + rr > h || start.y - rr < -h || start.y + rr > h;
    const bool col = real && dmax(0.0, norm(start - V2{xo, yo}) - ro) < rr;
    if (wall || __any_sync(kFull, col)) {
      *residual = 0.0;
      return 1;
    }
  }
  const V2 delta = (end - start) * (1.0 / C.substeps);
  const double max_diam = warp_max(real ? 2.0 * ro : 0.0);
  const double reach = (C.push_distance + C.tip_r) + 2.0 * max_diam;
  const unsigned active = __ballot_sync(kFull, real && dist_point_segment(V2{xo, yo}, start, end) <= reach + ro);
  const int P = n * (n - 1) / 2;
  const int nw = (P + 31) >> 5;
  // this lane's pairs (p = 32w + l), their squared reach and position caches
  int pi[kWarpWords], pj[kWarpWords];
  unsigned pact[kWarpWords];  // warp-uniform: active pairs per word
  double rs[kWarpWords], rr2[kWarpWords], ax[kWarpWords], ay[kWarpWords], bx[kWarpWords], by[kWarpWords];
#pragma unroll
  for (int w = 0; w < kWarpWords; ++w) {
    const int p = 32 * w + l;
    const bool valid = w < nw && p < P;
    const int ij = valid ? pij[p] : 0;
    pi[w] = ij & 0xff;
    pj[w] = ij >> 8;
    pact[w] = __ballot_sync(kFull, valid && (active >> pi[w] & 1u) && (active >> pj[w] & 1u));
    rs[w] = __shfl_sync(kFull, ro, pi[w]) + __shfl_sync(kFull, ro, pj[w]);  // br_a + br_b
    rr2[w] = rs[w] * rs[w];
    ax[w] = ay[w] = bx[w] = by[w] = 0.0;
  }
  const double hcl = C.side / 2.0 - C.margin - 1e-9;
  const bool mine = real && (active >> l & 1u);
  const double tr = C.tip_r;
  for (int step = 1; step <= C.substeps; ++step) {
    const V2 tc = start + delta * static_cast<double>(step);
    for (int iter = 0; iter < C.max_iters; ++iter) {
      double mp = 0.0;
      // tip vs own object (push_sim.cpp:90-100)
      if (mine) {
        const double dx = xo - tc.x, dy = yo - tc.y;
        const double d2 = dx * dx + dy * dy;
        const double rt = tr + ro;
        if (!(d2 > rt * rt)) {
          const double dist = sqrt(d2);
          const double depth = tr + ro - dist;
          if (depth > 0.0) {
            double ux = 1.0, uy = 0.0;
            if (dist > 0.0) {
              const double inv = __drcp_rn(dist);  // == 1.0 / dist
              ux = dx * inv;
              uy = dy * inv;
            }
            xo = xo + ux * depth;
            yo = yo + uy * depth;
            mp = depth;
          }
        }
      }
      // pair broad phase (push_sim.cpp:107-108) on refreshed caches
      unsigned cand[kWarpWords];
#pragma unroll
      for (int w = 0; w < kWarpWords; ++w) {
        cand[w] = 0u;
        if (w < nw) {  // warp-uniform
          ax[w] = __shfl_sync(kFull, xo, pi[w]);
          ay[w] = __shfl_sync(kFull, yo, pi[w]);
          bx[w] = __shfl_sync(kFull, xo, pj[w]);
          by[w] = __shfl_sync(kFull, yo, pj[w]);
          const double ex = ax[w] - bx[w], ey = ay[w] - by[w];
          cand[w] = __ballot_sync(kFull, (pact[w] >> l & 1u) && !(ex * ex + ey * ey > rr2[w]));
        }
      }
      // lexicographic candidate sweep (uniform); each set bit passes the
      // broad test on the current poses
#pragma unroll
      for (int w = 0; w < kWarpWords; ++w) {
        while (w < nw && cand[w]) {
          const int b = __ffs(cand[w]) - 1;
          cand[w] &= cand[w] - 1;
          const int p = 32 * w + b;
          const int ij = pij[p];
          const int i = ij & 0xff, j = ij >> 8;
          const double xi = __shfl_sync(kFull, xo, i), yi = __shfl_sync(kFull, yo, i);
          const double xj = __shfl_sync(kFull, xo, j), yj = __shfl_sync(kFull, yo, j);
          const double ri = __shfl_sync(kFull, ro, i), rj = __shfl_sync(kFull, ro, j);
          const double ex = xi - xj, ey = yi - yj;
          const double d2 = ex * ex + ey * ey;
          const double dist = sqrt(d2);  // == norm(pos_j - pos_i)
          const double depth = ri + rj - dist;
          if (depth > 0.0) {
            double ux = 1.0, uy = 0.0;
            if (dist > 0.0) {
              const double inv = __drcp_rn(dist);
              ux = (xj - xi) * inv;
              uy = (yj - yi) * inv;
            }
            const double s = 0.5 * depth;
            const double mx = ux * s, my = uy * s;
            const double nxi = xi - mx, nyi = yi - my, nxj = xj + mx, nyj = yj + my;
            if (l == i) {
              xo = nxi;
              yo = nyi;
            }
            if (l == j) {
              xo = nxj;
              yo = nyj;
            }
            mp = dmax(mp, depth);
            // patch the caches and re-test the later active pairs touching i or j
#pragma unroll
            for (int v = 0; v < kWarpWords; ++v) {
              if (v < w || v >= nw) continue;  // warp-uniform: only words holding pairs after p
              if (pi[v] == i) {
                ax[v] = nxi;
                ay[v] = nyi;
              } else if (pi[v] == j) {
                ax[v] = nxj;
                ay[v] = nyj;
              }
              if (pj[v] == i) {
                bx[v] = nxi;
                by[v] = nyi;
              } else if (pj[v] == j) {
                bx[v] = nxj;
                by[v] = nyj;
              }
              const int q = 32 * v + l;
              const bool touch = q > p && (pact[v] >> l & 1u) &&
                                 (pi[v] == i || pi[v] == j || pj[v] == i || pj[v] == j);
              const double fx = ax[v] - bx[v], fy = ay[v] - by[v];
              const bool pass = touch && !(fx * fx + fy * fy > rr2[v]);
              const unsigned tm = __ballot_sync(kFull, touch);
              const unsigned pm = __ballot_sync(kFull, pass);
              cand[v] = (cand[v] & ~tm) | pm;
            }
          }
        }
      }
      // clamp every object (push_sim.cpp:118 -> :48-54)
      if (real) {
        if (!(fabs(xo) <= hcl)) xo = fmin(fmax(xo, -hcl), hcl);
        if (!(fabs(yo) <= hcl)) yo = fmin(fmax(yo, -hcl), hcl);
      }
      if (!__any_sync(kFull, mp > C.eps_pen)) break;  // max_pen <= eps_pen
    }
  }
  // final all-pairs check (world.cpp:139-152), order-free max
  double worst = 0.0;
#pragma unroll
  for (int w = 0; w < kWarpWords; ++w) {
    if (w < nw) {
      const double fx = __shfl_sync(kFull, xo, pi[w]) - __shfl_sync(kFull, xo, pj[w]);
      const double fy = __shfl_sync(kFull, yo, pi[w]) - __shfl_sync(kFull, yo, pj[w]);
      const double d2 = fx * fx + fy * fy;
      if (32 * w + l < P && !(d2 > rr2[w])) worst = dmax(worst, rs[w] - sqrt(d2));  // (ra + rb) - dist
    }
  }
  worst = warp_max(worst);
  if (real) {
    W.x[l] = xo;
    W.y[l] = yo;
  }
  __syncwarp();
  *residual = worst;
  return worst > C.eps_pen ? 2 : 0;
}

// MT19937-64 twist of one env's 312-word block by a warp (three dependency
// phases of libstdc++ _M_gen_rand: k < 156 reads only old words; 156 <= k <
// 311 reads old k, k+1 and the NEW k-156; k = 311 reads new 0 and 155).
PPG_DI void warp_twist(const MtView& g, int l) {
  const uint64_t UM = 0xffffffff80000000ull, LM = 0x7fffffffull, A = 0xb5026f5aa96619e9ull;
  uint64_t nv[5];
#pragma unroll
  for (int t = 0; t < 5; ++t) {
    const int k = l + 32 * t;
    if (k < 156) {
      const uint64_t y = (g.w(k) & UM) | (g.w(k + 1) & LM);
      nv[t] = g.w(k + 156) ^ (y >> 1) ^ ((y & 1) ? A : 0);
    }
  }
  __syncwarp();
#pragma unroll
  for (int t = 0; t < 5; ++t) {
    const int k = l + 32 * t;
    if (k < 156) g.w(k) = nv[t];
  }
  __syncwarp();
#pragma unroll
  for (int t = 0; t < 5; ++t) {
    const int k = 156 + l + 32 * t;
    if (k < 311) {
      const uint64_t y = (g.w(k) & UM) | (g.w(k + 1) & LM);
      nv[t] = g.w(k - 156) ^ (y >> 1) ^ ((y & 1) ? A : 0);
    }
  }
  __syncwarp();
#pragma unroll
  for (int t = 0; t < 5; ++t) {
    const int k = 156 + l + 32 * t;
    if (k < 311) g.w(k) = nv[t];
  }
  __syncwarp();
  if (l == 0) {
    const uint64_t y = (g.w(311) & UM) | (g.w(0) & LM);
    g.w(311) = g.w(155) ^ (y >> 1) ^ ((y & 1) ? A : 0);
  }
  __syncwarp();
}

PPG_DI uint64_t warp_mt_next(const MtView& g, int& idx, int l) {
  if (idx >= 312) {
    warp_twist(g, l);
    idx = 0;
  }
  uint64_t z = g.w(idx++);
  z ^= (z >> 29) & 0x5555555555555555ull;
  z ^= (z << 17) & 0x71d67fffeda60000ull;
  z ^= (z << 37) & 0xfff7eee000000000ull;
  z ^= (z >> 43);
  return z;
}

// uniform_int_distribution<size_t>(0, n-1) (uniform_int_dist.h:255-280)
PPG_DI uint64_t warp_mt_pick(const MtView& g, int& idx, uint64_t n, int l) {
  uint64_t xw = warp_mt_next(g, idx, l);
  uint64_t low = xw * n, high = __umul64hi(xw, n);
  if (low < n) {
    const uint64_t thr = (0ull - n) % n;
    while (low < thr) {
      xw = warp_mt_next(g, idx, l);
      low = xw * n;
      high = __umul64hi(xw, n);
    }
  }
  return high;
}

// sample_pushes validity ballots; valid[w] bit b <=> candidate 32w+b is kept.
PPG_DI int warp_sample_mask(const WarpEnv& W, const ShapeView& S, const SimConst& C, unsigned* valid) {
  const int total = W.n * C.na;
  const int nw = (total + 31) >> 5;
  const PoseView P = W.view();
  int count = 0;
  for (int w = 0; w < nw; ++w) {
    const int c = 32 * w + W.lane;
    V2 s, t;
    const bool ok = c < total && push_candidate(P, S, C, c / C.na, c % C.na, true, s, t);
    const unsigned b = __ballot_sync(kFull, ok);
    if (W.lane == 0) valid[w] = b;
    count += __popc(b);
  }
  __syncwarp();
  return count;
}

// graspable over 16 lanes (one angle each) + ordered argmax.
PPG_DI GraspOut warp_graspable(const WarpEnv& W, const ShapeView& S, const SimConst& C, int target) {
  const int l = W.lane;
  double m = -1.0, cx = 0.0, cy = 0.0;
  bool f = false;
  if (l < kGraspAngles) f = grasp_angle(W.view(), S, C, target, l, &m, &cx, &cy);
  int k = f ? l : 1 << 20;
  if (!f) m = -1.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double om = __shfl_xor_sync(kFull, m, o);
    const int ok = __shfl_xor_sync(kFull, k, o);
    const double ox = __shfl_xor_sync(kFull, cx, o);
    const double oy = __shfl_xor_sync(kFull, cy, o);
    const bool take = om > m || (om == m && ok < k);
    if (take) {
      m = om;
      k = ok;
      cx = ox;
      cy = oy;
    }
  }
  GraspOut g{false, 0.0, 0.0, 0.0, -1};
  if (k < kGraspAngles) {
    g.k = k;
    g.margin = m;
    g.x = cx;
    g.y = cy;
    g.graspable = m >= C.margin_threshold;
  }
  return g;
}

}  // namespace

// ---------------------------------------------------------------------------

// batch_resolve, one warp per environment (small batches).
__global__ void __launch_bounds__(kWarpsPerBlock * 32) resolve_warp_kernel(const __grid_constant__ SimConst C,
                                                                          ResolveArgs a) {
  __shared__ double blk[kWarpsPerBlock][160];
  __shared__ uint16_t pij[kWarpMaxN * (kWarpMaxN - 1) / 2];
  build_pairs(pij, C.n);
  const int wib = threadIdx.x >> 5;
  const int e = blockIdx.x * kWarpsPerBlock + wib;
  const int E = a.E_dev ? *a.E_dev : a.E;
  if (e >= E) return;
  const int ee = a.idx ? a.idx[e] : e;
  WarpEnv W(blk[wib], C.n, static_cast<int>(threadIdx.x & 31));
  const ShapeView S = a.S.view(a.S.T == 1 ? 0 : ee);
  const int n = C.n;
  warp_load(W, a.poses_in + static_cast<size_t>(ee) * n * 3, S);
  const double* pu = a.pushes + static_cast<size_t>(ee) * 4;
  double residual = 0.0;
  const int st = warp_resolve(W, C, pij, V2{pu[0], pu[1]}, V2{pu[2], pu[3]}, true, &residual);
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
}

// batch_expand prepare (pmbs.cpp:82-93), one warp per (node, action) pair.
__global__ void __launch_bounds__(kWarpsPerBlock * 32) expand_warp_kernel(const __grid_constant__ SimConst C,
                                                                         ExpandArgs a) {
  __shared__ double blk[kWarpsPerBlock][160];
  __shared__ unsigned valid[kWarpsPerBlock][32];
  __shared__ uint16_t pij[kWarpMaxN * (kWarpMaxN - 1) / 2];
  build_pairs(pij, C.n);
  const int wib = threadIdx.x >> 5;
  const int p = blockIdx.x * kWarpsPerBlock + wib;
  if (p >= a.P) return;
  const int n = C.n, l = threadIdx.x & 31;
  WarpEnv W(blk[wib], n, l);
  const ShapeView S = a.S.view(0);
  const double* parent = a.parent_poses + static_cast<size_t>(p) * n * 3;
  warp_load(W, parent, S);
  const double* act = a.actions + static_cast<size_t>(p) * 4;
  double residual;
  const int st = warp_resolve(W, C, pij, V2{act[0], act[1]}, V2{act[2], act[3]}, true, &residual);
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
__global__ void __launch_bounds__(kWarpsPerBlock * 32) lock_step_warp_kernel(const __grid_constant__ SimConst C,
                                                                            LockArgs a) {
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
  warp_load(W, env, S);
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
  const int st = warp_resolve(W, C, pij, s, t, false, &residual);
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

}  // namespace ppg
