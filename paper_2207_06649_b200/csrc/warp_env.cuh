// warp_env.cuh — latency mode: ONE WARP PER ENVIRONMENT (disc scenes, n <= 23).
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
//  * pair phase (push_sim.cpp:101-117): pair p is owned by lane p % 32;
//    ballots give warp-uniform candidate / hit masks walked in lexicographic
//    order; after a hit on (i,j) the lanes owning LATER pairs touching i or j
//    re-evaluate them on the new poses, so every set bit always means what
//    the reference's in-place Gauss-Seidel sweep sees when it reaches that
//    pair (warp_resolve below has the two variants);
//  * the convergence test max_pen <= eps (push_sim.cpp:119) is a ballot;
//  * sample_pushes (actions.cpp:51-73): candidate c tested by lane c % 32,
//    validity ballots give the (object, angle)-ordered list;
//  * graspable (actions.cpp:113-147): lane k evaluates grasp angle k; the
//    first strict maximum in index order == max margin, lowest k on ties;
//  * MT19937-64: the 312-word block twist runs on 32 lanes in its three
//    dependency phases (libstdc++ _M_gen_rand).
//
// Poses live in shared memory (per-warp block x[n] | y[n] | theta[n], radii
// at +128); every max reduction is over non-negative values starting at +0.0,
// so its result does not depend on the order.
#pragma once

#include <cuda_runtime.h>

#include "kernels.cuh"

namespace ppg {

constexpr int kWarpMaxN = 23;   // pair masks: 8 ballot words (253 pairs)
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

// Pair-mask words (32 pairs each) for n objects: the resolve below is
// instantiated per word count so every loop over words is unrolled with no
// run-time guards.
PPG_HD constexpr int warp_words_for(int n) { return n <= 8 ? 1 : n <= 11 ? 2 : n <= 16 ? 4 : 8; }

// resolve_push (push_sim.cpp:58-130) for a disc scene, one warp.  Returns
// 0 ok, 1 start collision, 2 not converged (uniform); *residual = final max
// pairwise penetration.
//
// The per-warp shared block (W.x, W.y) is the single copy of the positions.
// Lane l owns object l in the tip phase (objects are independent there) and
// the clamp, and pairs p = 32w + l (w < NW) in the pair phase.  The pair
// phase is the reference's in-place Gauss-Seidel sweep in lexicographic
// order (push_sim.cpp:101-117), restated so that every pair is evaluated on
// exactly the positions the sweep sees when it reaches it:
//
//  * NW <= 2 (n <= 11, the paper's scenes) — speculative: each lane
//    evaluates its pairs' broad + narrow test at once (pair_eval); the sweep
//    walks the hits in order, the owner lane applies a hit (two stores) and
//    only the lanes holding LATER pairs touching the two moved objects
//    re-evaluate theirs.  The serial chain per hit is one re-evaluation.
//  * NW >= 4 (dense scenes) — uniform: the broad test is a ballot per word,
//    the candidates' narrow tests run uniformly across the warp (broadcast
//    loads), and after a hit only the later pairs touching the moved objects
//    re-run their broad test.  Fewer FP64 instructions per hit when a word
//    holds many touched pairs.
// A candidate whose narrow test finds no overlap changes nothing, so the
// speculative variant keeps hit masks only.
// One disc pair's broad + narrow phase (push_sim.cpp:107-108; disc_disc_
// overlap geometry.cpp:107-115 via object_pair_overlap push_sim.cpp:20-32)
// evaluated speculatively by the lane that owns the pair, on the current
// positions.  Returns "hit" (broad test passes and depth > 0); for a hit,
// depth and the two moved positions (apply_contact_motion with -/+ half the
// depth, :36-46) are the reference's values.  Branch-free, so the chains of
// a lane's pairs in different words overlap; `live` = the lane evaluates
// this pair — other lanes take a benign d2 = 1 so no lane enters the sqrt /
// reciprocal special-case paths (d2 = 0 for the padding pairs).
PPG_DI bool pair_eval_bf(const double* X, const double* Y, int a, int b, double rr2, double rsum, bool live,
                         double& nxa, double& nya, double& nxb, double& nyb, double& depth) {
  const double xa = X[a], ya = Y[a], xb = X[b], yb = Y[b];
  const double ex = xa - xb, ey = ya - yb;
  const double d2 = live ? ex * ex + ey * ey : 1.0;
  const double dist = sqrt(d2);  // == norm(pos_b - pos_a)
  depth = rsum - dist;
  const bool pos = dist > 0.0;
  const double inv = __drcp_rn(pos ? dist : 1.0);  // == 1.0 / dist
  const double ux = pos ? (xb - xa) * inv : 1.0;
  const double uy = pos ? (yb - ya) * inv : 0.0;
  const double s = 0.5 * depth;
  const double mx = ux * s, my = uy * s;
  nxa = xa - mx;
  nya = ya - my;
  nxb = xb + mx;
  nyb = yb + my;
  return !(d2 > rr2) && depth > 0.0;
}

// The branched form of pair_eval_bf (early exits; same results).
PPG_DI bool pair_eval(const double* X, const double* Y, int a, int b, double rr2, double rsum, double& nxa,
                      double& nya, double& nxb, double& nyb, double& depth) {
  const double xa = X[a], ya = Y[a], xb = X[b], yb = Y[b];
  const double ex = xa - xb, ey = ya - yb;
  const double d2 = ex * ex + ey * ey;
  depth = 0.0;
  if (d2 > rr2) return false;
  const double dist = sqrt(d2);  // == norm(pos_b - pos_a)
  depth = rsum - dist;
  if (!(depth > 0.0)) return false;
  double ux = 1.0, uy = 0.0;
  if (dist > 0.0) {
    const double inv = __drcp_rn(dist);  // == 1.0 / dist
    ux = (xb - xa) * inv;
    uy = (yb - ya) * inv;
  }
  const double s = 0.5 * depth;
  const double mx = ux * s, my = uy * s;
  nxa = xa - mx;
  nya = ya - my;
  nxb = xb + mx;
  nyb = yb + my;
  return true;
}

template <int NW>
PPG_DI int warp_resolve(WarpEnv& W, const SimConst& C, const uint16_t* pij, V2 start, V2 end, bool check_start,
                        double* residual) {
  constexpr bool kSpec = NW <= 2;
  const int n = W.n, l = W.lane;
  double* X = W.x;
  double* Y = W.y;
  const double* R = W.r;
  __syncwarp();
  const bool real = l < n;
  double xo = real ? X[l] : 0.0, yo = real ? Y[l] : 0.0;
  const double ro = real ? R[l] : 0.0;
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
  // this lane's pairs p = 32w + l: objects, object bitmask (0 = inactive
  // pair), squared reach; speculative narrow-phase results
  int pa[NW], pb[NW];
  unsigned om[NW];
  double rs[NW], rr2[NW];
  double nxa[NW], nya[NW], nxb[NW], nyb[NW], dep[NW];
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const int p = 32 * w + l;
    const bool valid = p < P;
    const int ij = valid ? pij[p] : 0;
    pa[w] = ij & 0xff;
    pb[w] = ij >> 8;
    const bool act = valid && (active >> pa[w] & 1u) && (active >> pb[w] & 1u);
    om[w] = act ? (1u << pa[w]) | (1u << pb[w]) : 0u;
    rs[w] = R[pa[w]] + R[pb[w]];  // br_a + br_b
    rr2[w] = rs[w] * rs[w];
    nxa[w] = nya[w] = nxb[w] = nyb[w] = dep[w] = 0.0;
  }
  const double hcl = C.side / 2.0 - C.margin - 1e-9;
  const bool mine = real && (active >> l & 1u);
  const double tr = C.tip_r;
  for (int step = 1; step <= C.substeps; ++step) {
    const V2 tc = start + delta * static_cast<double>(step);
    for (int iter = 0; iter < C.max_iters; ++iter) {
      double mp = 0.0;  // this lane's part of max_pen (order-free max)
      const double xs = kSpec ? 0.0 : xo, ys = kSpec ? 0.0 : yo;  // own object at the iteration start
      // tip vs own object (push_sim.cpp:90-100)
      {  // branch-free; lanes without an active object take benign inputs
        const double dx = xo - tc.x, dy = yo - tc.y;
        const double d2r = dx * dx + dy * dy;
        const double rt = tr + ro;
        const bool near = mine && !(d2r > rt * rt);
        const double dist = sqrt(near ? d2r : 1.0);
        const double depth = tr + ro - dist;
        const bool pos = dist > 0.0;
        const double inv = __drcp_rn(pos ? dist : 1.0);  // == 1.0 / dist
        const double ux = pos ? dx * inv : 1.0, uy = pos ? dy * inv : 0.0;
        if (near && depth > 0.0) {
          xo = xo + ux * depth;
          yo = yo + uy * depth;
          X[l] = xo;
          Y[l] = yo;
          mp = depth;
        }
      }
      __syncwarp();
      if constexpr (kSpec) {
        unsigned hit[NW];
        // every word's chain side by side, branch-free
        bool h[NW];
#pragma unroll
        for (int w = 0; w < NW; ++w)
          h[w] = pair_eval_bf(X, Y, pa[w], pb[w], rr2[w], rs[w], om[w] != 0u, nxa[w], nya[w], nxb[w], nyb[w], dep[w]) &&
                 om[w] != 0u;
#pragma unroll
        for (int w = 0; w < NW; ++w) hit[w] = __ballot_sync(kFull, h[w]);
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          while (hit[w]) {
            const int b = __ffs(hit[w]) - 1;
            hit[w] &= hit[w] - 1;
            const unsigned hm = __shfl_sync(kFull, om[w], b);
            __syncwarp();  // every lane is done reading the old positions
            if (l == b) {
              X[pa[w]] = nxa[w];
              Y[pa[w]] = nya[w];
              X[pb[w]] = nxb[w];
              Y[pb[w]] = nyb[w];
              mp = dmax(mp, dep[w]);
            }
            __syncwarp();
            if constexpr (NW == 2) {
              if (w == 0) {
                // both words: the two re-tests are independent chains, run
                // branch-free side by side (a lane keeps its old results
                // where it does not re-test)
                const bool t0 = (om[0] & hm) != 0u && l > b;
                const bool t1 = (om[1] & hm) != 0u;
                double a0, a1, a2, a3, a4, c0, c1, c2, c3, c4;
                const bool h0 = pair_eval_bf(X, Y, pa[0], pb[0], rr2[0], rs[0], t0, a0, a1, a2, a3, a4);
                const bool h1 = pair_eval_bf(X, Y, pa[1], pb[1], rr2[1], rs[1], t1, c0, c1, c2, c3, c4);
                if (t0) {
                  nxa[0] = a0;
                  nya[0] = a1;
                  nxb[0] = a2;
                  nyb[0] = a3;
                  dep[0] = a4;
                }
                if (t1) {
                  nxa[1] = c0;
                  nya[1] = c1;
                  nxb[1] = c2;
                  nyb[1] = c3;
                  dep[1] = c4;
                }
                const unsigned tm0 = __ballot_sync(kFull, t0), tm1 = __ballot_sync(kFull, t1);
                hit[0] = (hit[0] & ~tm0) | __ballot_sync(kFull, t0 && h0);
                hit[1] = (hit[1] & ~tm1) | __ballot_sync(kFull, t1 && h1);
                continue;
              }
            }
            // w is the last word here: only its later pairs touching the
            // moved objects are re-tested — branch-free for one word (n <= 8,
            // measured 15 % faster), branched for the second of two words
            // (the branch skips the re-test when no lane holds one)
            if constexpr (NW == 2) {
              const bool t = (om[w] & hm) != 0u && l > b;
              bool h = false;
              if (t) h = pair_eval(X, Y, pa[w], pb[w], rr2[w], rs[w], nxa[w], nya[w], nxb[w], nyb[w], dep[w]);
              const unsigned tm = __ballot_sync(kFull, t);
              hit[w] = (hit[w] & ~tm) | __ballot_sync(kFull, h);
            } else {
              const bool t = (om[w] & hm) != 0u && l > b;
              double a0, a1, a2, a3, a4;
              const bool h = pair_eval_bf(X, Y, pa[w], pb[w], rr2[w], rs[w], t, a0, a1, a2, a3, a4);
              if (t) {
                nxa[w] = a0;
                nya[w] = a1;
                nxb[w] = a2;
                nyb[w] = a3;
                dep[w] = a4;
              }
              const unsigned tm = __ballot_sync(kFull, t);
              hit[w] = (hit[w] & ~tm) | __ballot_sync(kFull, t && h);
            }
          }
        }
      } else {
        // broad phase ballots
        unsigned cand[NW];
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          const double ex = X[pa[w]] - X[pb[w]], ey = Y[pa[w]] - Y[pb[w]];
          cand[w] = __ballot_sync(kFull, om[w] != 0u && !(ex * ex + ey * ey > rr2[w]));
        }
        // uniform lexicographic candidate sweep
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          while (cand[w]) {
            const int b = __ffs(cand[w]) - 1;
            cand[w] &= cand[w] - 1;
            const int p = 32 * w + b;
            const int ij = pij[p];
            const int i = ij & 0xff, j = ij >> 8;
            const double xi = X[i], yi = Y[i], xj = X[j], yj = Y[j];
            const double ex = xi - xj, ey = yi - yj;
            const double d2 = ex * ex + ey * ey;
            const double dist = sqrt(d2);  // == norm(pos_j - pos_i)
            const double depth = R[i] + R[j] - dist;
            if (depth > 0.0) {
              double ux = 1.0, uy = 0.0;
              if (dist > 0.0) {
                const double inv = __drcp_rn(dist);
                ux = (xj - xi) * inv;
                uy = (yj - yi) * inv;
              }
              const double s = 0.5 * depth;
              const double mx = ux * s, my = uy * s;
              __syncwarp();  // every lane has read the old positions
              if (l == 0) {
                X[i] = xi - mx;
                Y[i] = yi - my;
                X[j] = xj + mx;
                Y[j] = yj + my;
              }
              __syncwarp();
              mp = dmax(mp, depth);
              // re-test the later active pairs touching i or j: every word's
              // broad test side by side (independent, branch-free), then the
              // votes
              const unsigned hm = (1u << i) | (1u << j);
              bool touch[NW], pass[NW];
#pragma unroll
              for (int v = 0; v < NW; ++v) {
                touch[v] = v >= w && (om[v] & hm) != 0u && 32 * v + l > p;
                const double fx = X[pa[v]] - X[pb[v]], fy = Y[pa[v]] - Y[pb[v]];
                pass[v] = touch[v] && !(fx * fx + fy * fy > rr2[v]);
              }
#pragma unroll
              for (int v = w; v < NW; ++v) {
                const unsigned tm = __ballot_sync(kFull, touch[v]);
                cand[v] = (cand[v] & ~tm) | __ballot_sync(kFull, pass[v]);
              }
            }
          }
        }
      }
      // clamp every object (push_sim.cpp:118 -> :48-54)
      if (real) {
        xo = X[l];
        yo = Y[l];
        if (!(fabs(xo) <= hcl)) X[l] = xo = fmin(fmax(xo, -hcl), hcl);
        if (!(fabs(yo) <= hcl)) Y[l] = yo = fmin(fmax(yo, -hcl), hcl);
      }
      if (!__any_sync(kFull, mp > C.eps_pen)) break;  // max_pen <= eps_pen
      // Fixed point: this iteration left every position bit-identical, so
      // each remaining iteration of the substep repeats it exactly (same
      // state, same tip position, same max_pen > eps) up to max_iters:
      // skipping them gives the same state (jammed pushes, ~87 % of the
      // iterations that exhaust max_iters in rollouts).
      // (dense scenes only: for n <= 11 the check's code costs more than the
      // skipped iterations save — measured 5 % slower on case_18 at N_e = 64)
      if constexpr (!kSpec)
        if (C.fixpoint && __all_sync(kFull, __double_as_longlong(xo) == __double_as_longlong(xs) &&
                                                  __double_as_longlong(yo) == __double_as_longlong(ys)))
          break;
    }
  }
  // final all-pairs check (world.cpp:139-152), order-free max
  __syncwarp();
  double worst = 0.0;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const double fx = X[pa[w]] - X[pb[w]], fy = Y[pa[w]] - Y[pb[w]];
    const double d2 = fx * fx + fy * fy;
    if (32 * w + l < P && !(d2 > rr2[w])) worst = dmax(worst, rs[w] - sqrt(d2));  // (ra + rb) - dist
  }
  worst = warp_max(worst);
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

constexpr int kMtFrozen = 1 << 20;  // idx after a frozen view needed a twist

PPG_DI uint64_t warp_mt_next(const MtView& g, int& idx, int l) {
  if (idx >= 312) {
    if (g.frozen) {  // the state must stay untouched: abort the draw
      idx = kMtFrozen;
      return 0;
    }
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
  if (idx >= kMtFrozen) return 0;
  uint64_t low = xw * n, high = __umul64hi(xw, n);
  if (low < n) {
    const uint64_t thr = (0ull - n) % n;
    while (low < thr) {
      xw = warp_mt_next(g, idx, l);
      if (idx >= kMtFrozen) return 0;
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

}  // namespace ppg
