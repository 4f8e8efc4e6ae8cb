// warp_poly.cuh — latency mode for scenes WITH POLYGONS: resolve_push
// (push_sim.cpp:58-130) by one warp per environment, n <= 16, bit-exact.
//
// The generic one-lane resolve spends a polygon narrow test in a long serial
// chain (14 SAT axes, each with a sqrt + two divisions and two support
// scans; closest points over every edge).  Here the warp evaluates one
// narrow test at a time (the candidates are still taken in the reference's
// lexicographic Gauss-Seidel order) with the work spread over lanes:
//
//  * polygon_polygon_overlap (geometry.cpp:156-174): lane k < |A| evaluates
//    axis k of sat_min_overlap(A, B), lane 16 + k axis k of
//    sat_min_overlap(B, A).  The reference's early exit returns "separated"
//    iff some axis of the first (then the second) call has o <= 0, and the
//    overlap depth is the FIRST strict minimum over the axes in that order:
//    a ballot and a (value, lane) min-reduction reproduce both exactly.  A
//    separated pair changes nothing (depth <= 0 is never applied), so its
//    negative depth is not computed (same decisions, same bits).
//  * closest_point_on_polygon (geometry.cpp:87-100): lane k evaluates edge
//    k; first strict minimum of the squared distance = (value, lane) min.
//    The contact of a polygon pair runs both closest-point scans at once in
//    the two half-warps.  point_in_convex is a ballot.
//  * world polygons (world.cpp:57-62) and centroids (geometry.cpp:66-79) are
//    CACHED per object in shared memory and refreshed whenever the object's
//    pose changes: world_polygon is a pure function of (x, y, theta) with
//    theta's glibc sincos (glibc_sincos.cuh), so the cache is bit-identical
//    to the reference's per-test recomputation.
//  * the tip phase (objects independent, push_sim.cpp:90-100), the clamp and
//    the final penetration check run one object / one pair per lane with the
//    scalar geometry of geom.cuh on the cached polygons.
#pragma once

#include "warp_env.cuh"

namespace ppg {

constexpr int kPolyMaxN = 16;  // polygon latency mode: objects per scene

namespace {

// Code size matters here: with the narrow-phase body inlined once per
// pair-mask word (and the contact motion, which holds a sincos, twice per
// hit) the kernels grew past 500 KB of SASS and stalled on instruction fetch
// (ncu: "no_instruction" 59 % of the cycles between issues, polygon
// batch_resolve at 0.73 M env-steps/s).  The candidate sweep and the motion
// are now loops emitting each body once (2.1 M env-steps/s); the final check
// is out of line.
#define PPG_NI __device__ __noinline__

// Per-warp polygon caches (shared memory).
struct WarpPoly {
  V2* wv;   // [kPolyMaxN][kMaxV] world vertices
  V2* cen;  // [kPolyMaxN] centroids
};

struct PolyShape {  // this lane's object (lane l < n)
  int kind, nv;
  double r, br;
};

PPG_DI void lane_poly(const WarpPoly& G, int i, int nv, Poly& out) {
  out.n = nv;
#pragma unroll
  for (int k = 0; k < kMaxV; ++k)
    if (k < nv) out.p[k] = G.wv[i * kMaxV + k];
}

// world_polygon + polygon_centroid of object i, computed by ONE lane.
PPG_DI void lane_refresh(const WarpEnv& W, const WarpPoly& G, const ShapeView& S, int i, int nv) {
  const double s = W.view().s(i), c = W.view().c(i);
  const V2 pos{W.x[i], W.y[i]};
  PPG_ROLLED
  for (int k = 0; k < nv; ++k) {
    const V2 v = S.vert(i, k);
    G.wv[i * kMaxV + k] = pos + V2{c * v.x - s * v.y, s * v.x + c * v.y};
  }
  G.cen[i] = polygon_centroid(PolyRef{G.wv + i * kMaxV, nv});
}

// Loads the trig cache and the world polygons of every polygon object (lane
// per object); called after warp_load.
PPG_DI PolyShape warp_poly_load(const WarpEnv& W, const WarpPoly& G, const ShapeView& S) {
  const int l = W.lane;
  PolyShape o{0, 0, 0.0, 0.0};
  if (l < W.n) {
    o.kind = S.kind_(l);
    o.r = S.rad_(l);
    o.br = S.br_(l);
    o.nv = o.kind != 0 ? S.nv_(l) : 0;
    if (o.kind != 0) {
      double s, c;
      glibc_sincos(W.th[l], &s, &c);
      W.view().s(l) = s;
      W.view().c(l) = c;
      lane_refresh(W, G, S, l, o.nv);
    }
  }
  __syncwarp();
  return o;
}

// (value, lane) minimum over the lanes in `mask` of a 16-lane half (off <=
// 8) or the whole warp (off <= 16): the first strict minimum in lane order.
PPG_DI void argmin_first(double& v, int& k, int top) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    if (o > top) continue;
    const double ov = __shfl_xor_sync(kFull, v, o);
    const int ok = __shfl_xor_sync(kFull, k, o);
    if (ov < v || (ov == v && ok < k)) {
      v = ov;
      k = ok;
    }
  }
}

// closest_point_on_polygon(p, poly) of the cached polygon `i` (nv edges),
// lanes base .. base + nv - 1, reduced within a half-warp (top = 8) or the
// full warp (top = 16).  Returns the point (valid in every lane of the
// half / warp).
PPG_DI V2 warp_closest(const WarpPoly& G, int i, int nv, V2 p, int base, int top, int l) {
  const int k = l - base;
  double d = inf_d();
  int key = 64 + l;
  V2 q{0.0, 0.0};
  if (k >= 0 && k < nv) {
    q = closest_point_on_segment(p, G.wv[i * kMaxV + k], G.wv[i * kMaxV + (k + 1 == nv ? 0 : k + 1)]);
    d = norm2(p - q);
    key = k;
  }
  double bd = d;
  int bk = key;
  argmin_first(bd, bk, top);
  const int src = base + (bk < 64 ? bk : 0);  // lane holding the winning edge
  return V2{__shfl_sync(kFull, q.x, src), __shfl_sync(kFull, q.y, src)};
}

// disc_polygon_overlap (geometry.cpp:117-132), uniform result.
PPG_DI Overlap warp_disc_poly(const WarpPoly& G, int i, int nv, V2 c, double r, int l) {
  const V2 q = warp_closest(G, i, nv, c, 0, 16, l);
  bool out = false;
  if (l < nv) {
    const V2 a = G.wv[i * kMaxV + l], b = G.wv[i * kMaxV + (l + 1 == nv ? 0 : l + 1)];
    out = cross(b - a, c - a) < 0.0;
  }
  const bool inside = !__any_sync(kFull, out);
  Overlap o;
  const V2 d = q - c;
  const double dist = norm(d);
  o.contact = q;
  o.depth = inside ? r + dist : r - dist;
  o.dir = dist > 0.0 ? d * (1.0 / dist) : V2{1.0, 0.0};
  return o;
}

// polygon_polygon_overlap (geometry.cpp:156-174), uniform result; *hit =
// overlapping (when false the depth is a non-positive placeholder).
PPG_DI Overlap warp_poly_poly(const WarpPoly& G, int a, int na, int b, int nb, int l, bool* hit) {
  // lane k < na: axis k of sat_min_overlap(A, B); lane 16 + k: axis k of (B, A)
  const bool first = l < 16;
  const int k = first ? l : l - 16;
  const int p = first ? a : b, q = first ? b : a;
  const int np = first ? na : nb, nq = first ? nb : na;
  const bool mine = k < np;
  double o = inf_d();
  V2 normal{0.0, 0.0};
  if (mine) {
    const V2 e = G.wv[p * kMaxV + (k + 1 == np ? 0 : k + 1)] - G.wv[p * kMaxV + k];
    normal = normalized(V2{e.y, -e.x});
    double pmax = -inf_d(), qmax = -inf_d();
    for (int t = 0; t < np; ++t) pmax = dmax(pmax, dot(G.wv[p * kMaxV + t], normal));
    const V2 nn = -normal;
    for (int t = 0; t < nq; ++t) qmax = dmax(qmax, dot(G.wv[q * kMaxV + t], nn));
    o = pmax - -qmax;  // a_max - b_min, b_min = -support_extent(b, -normal)
  }
  const unsigned sep = __ballot_sync(kFull, mine && o <= 0.0);
  if (o != o) o = inf_d();  // a NaN axis never becomes the depth (o < depth is false)
  Overlap r;
  r.contact = V2{0.0, 0.0};
  r.dir = V2{0.0, 0.0};
  if ((sep & 0xffffu) || (sep >> 16)) {  // the first call, else the second, found a separating axis
    *hit = false;
    r.depth = -0.0;
    return r;
  }
  double bo = o;
  int bk = mine ? l : 64 + l;
  argmin_first(bo, bk, 16);
  const V2 axis{__shfl_sync(kFull, normal.x, bk), __shfl_sync(kFull, normal.y, bk)};
  r.depth = bo;
  const V2 cb = G.cen[b], ca = G.cen[a];
  const V2 sepv = cb - ca;
  r.dir = dot(sepv, axis) >= 0.0 ? axis : -axis;
  // closest_point_on_polygon(cb, A) in lanes 0..na-1, (ca, B) in 16..16+nb-1
  const int hi = l & 16;
  const V2 qa = warp_closest(G, hi ? b : a, hi ? nb : na, hi ? ca : cb, hi, 8, l);
  const V2 qA{__shfl_sync(kFull, qa.x, 0), __shfl_sync(kFull, qa.y, 0)};
  const V2 qB{__shfl_sync(kFull, qa.x, 16), __shfl_sync(kFull, qa.y, 16)};
  r.contact = (qA + qB) * 0.5;
  *hit = true;
  return r;
}

// apply_contact_motion (push_sim.cpp:36-46) of object i, computed uniformly
// by the warp (every lane holds the same values); lane 0 stores the pose,
// the polygon cache is refreshed (vertex k by lane k).
PPG_DI void warp_apply_motion(const WarpEnv& W, const WarpPoly& G, const ShapeView& S, int i, int kind, int nv,
                              V2 t, V2 contact, double gain, int l) {
  const PoseView P = W.view();
  const double x = P.x(i) + t.x, y = P.y(i) + t.y;
  double th = P.th(i), c = 0.0, s = 0.0;
  bool rot = false;
  if (kind == 1 && gain != 0.0) {
    const V2 lever = contact - V2{x, y};
    const double lever2 = norm2(lever);
    if (!(lever2 < 1e-12)) {
      double dtheta = gain * cross(lever, t) / lever2;
      dtheta = dclamp(dtheta, -0.2, 0.2);
      th = wrap_angle(th + dtheta);
      glibc_sincos(th, &s, &c);
      rot = true;
    }
  }
  if (kind != 0 && !rot) {
    c = P.c(i);
    s = P.s(i);
  }
  __syncwarp();  // every lane is done reading the old pose / polygon
  if (l == 0) {
    P.x(i) = x;
    P.y(i) = y;
    if (rot) {
      P.th(i) = th;
      P.c(i) = c;
      P.s(i) = s;
    }
  }
  if (kind != 0 && l < nv) {
    const V2 v = S.vert(i, l);
    G.wv[i * kMaxV + l] = V2{x, y} + V2{c * v.x - s * v.y, s * v.x + c * v.y};
  }
  __syncwarp();
  if (kind != 0) {
    const V2 cen = polygon_centroid(PolyRef{G.wv + i * kMaxV, nv});  // identical in every lane
    __syncwarp();
    if (l == 0) G.cen[i] = cen;
    __syncwarp();
  }
}

// Narrow test of candidate pair ij (object_pair_overlap, push_sim.cpp:20-32)
// and, on a hit, the half-depth contact motion of both objects
// (push_sim.cpp:109-116); uniform over the warp.  Returns the hit's object
// mask (0: no hit) and raises *mp to the depth.
PPG_DI unsigned warp_pair_poly(const WarpEnv& W, const WarpPoly& G, const PolyShape& O, const ShapeView& S,
                               const SimConst& C, int ij, int l, double* mp) {
  const int i = ij & 0xff, j = ij >> 8;
  const int ki = __shfl_sync(kFull, O.kind, i), kj = __shfl_sync(kFull, O.kind, j);
  const int ni = __shfl_sync(kFull, O.nv, i), nj = __shfl_sync(kFull, O.nv, j);
  const double ri = __shfl_sync(kFull, O.r, i), rj = __shfl_sync(kFull, O.r, j);
  const V2 pi_{W.x[i], W.y[i]}, pj_{W.x[j], W.y[j]};
  Overlap o;
  bool hit;
  if (ki == 0 && kj == 0) {
    o = disc_disc_overlap(pi_, ri, pj_, rj);
    hit = o.depth > 0.0;
  } else if (ki == 0) {
    o = warp_disc_poly(G, j, nj, pi_, ri, l);
    hit = o.depth > 0.0;
  } else if (kj == 0) {
    o = warp_disc_poly(G, i, ni, pj_, rj, l);
    o.dir = -o.dir;
    hit = o.depth > 0.0;
  } else {
    o = warp_poly_poly(G, i, ni, j, nj, l, &hit);
    hit = hit && o.depth > 0.0;
  }
  if (!hit) return 0u;
  // i then j (one copy of the motion code: it holds a sincos)
#pragma unroll 1
  for (int side = 0; side < 2; ++side) {
    const bool si = side == 0;
    const V2 t = o.dir * (si ? -(0.5 * o.depth) : 0.5 * o.depth);
    warp_apply_motion(W, G, S, si ? i : j, si ? ki : kj, si ? ni : nj, t, o.contact, C.gain, l);
  }
  *mp = dmax(*mp, o.depth);
  return (1u << i) | (1u << j);
}

// Scalar object_pair_overlap depth (push_sim.cpp:20-32) on the caches, for
// the final penetration check (one pair per lane).
PPG_NI double lane_pair_depth(const WarpEnv& W, const WarpPoly& G, int a, int ka, int na, double ra, int b, int kb,
                              int nb, double rb) {
  const V2 pa{W.x[a], W.y[a]}, pb{W.x[b], W.y[b]};
  if (ka == 0 && kb == 0) return disc_disc_overlap(pa, ra, pb, rb).depth;
  if (ka == 0) return disc_polygon_overlap(pa, ra, PolyRef{G.wv + b * kMaxV, nb}).depth;
  if (kb == 0) return disc_polygon_overlap(pb, rb, PolyRef{G.wv + a * kMaxV, na}).depth;
  Poly A, B;
  lane_poly(G, a, na, A);
  lane_poly(G, b, nb, B);
  return polygon_polygon_overlap(A, B, false).depth;
}

// resolve_push for a scene with polygons, one warp (n <= 16).  Returns 0 ok,
// 1 start collision, 2 not converged (uniform); *residual = final max
// pairwise penetration.  W's pose block and G's caches must be loaded
// (warp_load + warp_poly_load); `O` is this lane's object.
template <int NW>
PPG_DI int warp_resolve_poly(WarpEnv& W, const WarpPoly& G, const PolyShape& O, const ShapeView& S,
                             const SimConst& C, const uint16_t* pij, V2 start, V2 end, bool check_start,
                             double* residual) {
  const int n = W.n, l = W.lane;
  double* X = W.x;
  double* Y = W.y;
  const PoseView P = W.view();
  __syncwarp();
  const bool real = l < n;
  // per-object shape scalars of every object, for the uniform narrow phase
  // (object j's values live in lane j)
  if (check_start) {  // collides_gripper_start (world.cpp:154-164) via object_point_distance (:101-107)
    const double rr = C.tip_r + C.tip_clear;
    const double h = C.side / 2.0;
    const bool wall = start.x - rr < -h || start.x + rr > h || start.y - rr < -h || start.y + rr > h;
    bool col = false;
    if (real) {
      double d;
      if (O.kind == 0) {
        d = dmax(0.0, norm(start - V2{X[l], Y[l]}) - O.r);
      } else {
        d = dmax(0.0, signed_dist_point_polygon(start, PolyRef{G.wv + l * kMaxV, O.nv}));
      }
      col = d < rr;
    }
    if (wall || __any_sync(kFull, col)) {
      *residual = 0.0;
      return 1;
    }
  }
  const V2 delta = (end - start) * (1.0 / C.substeps);
  const double max_diam = warp_max(real ? 2.0 * O.br : 0.0);
  const double reach = (C.push_distance + C.tip_r) + 2.0 * max_diam;
  const unsigned active =
      __ballot_sync(kFull, real && dist_point_segment(V2{X[l], Y[l]}, start, end) <= reach + O.br);
  const int Pn = n * (n - 1) / 2;
  int pa[NW], pb[NW];
  unsigned om[NW];
  double rr2[NW];
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const int p = 32 * w + l;
    const bool valid = p < Pn;
    const int ij = valid ? pij[p] : 0;
    pa[w] = ij & 0xff;
    pb[w] = ij >> 8;
    const bool act = valid && (active >> pa[w] & 1u) && (active >> pb[w] & 1u);
    om[w] = act ? (1u << pa[w]) | (1u << pb[w]) : 0u;
    const double rs = __shfl_sync(kFull, O.br, pa[w]) + __shfl_sync(kFull, O.br, pb[w]);  // br_a + br_b
    rr2[w] = rs * rs;
  }
  const double hcl = C.side / 2.0 - C.margin - 1e-9;
  const bool mine = real && (active >> l & 1u);
  const double tr = C.tip_r;
  for (int step = 1; step <= C.substeps; ++step) {
    const V2 tc = start + delta * static_cast<double>(step);
    for (int iter = 0; iter < C.max_iters; ++iter) {
      double mp = 0.0;
      const double xs = real ? X[l] : 0.0, ys = real ? Y[l] : 0.0, ts = real ? P.th(l) : 0.0;  // iteration start
      // tip vs own object (push_sim.cpp:90-100), lane per object
      if (mine) {
        const V2 pos{X[l], Y[l]};
        const double rt = tr + O.br;
        if (!(norm2(pos - tc) > rt * rt)) {
          Overlap o;
          if (O.kind == 0) {
            o = disc_disc_overlap(tc, tr, pos, O.r);
          } else {
            o = disc_polygon_overlap(tc, tr, PolyRef{G.wv + l * kMaxV, O.nv});
          }
          if (o.depth > 0.0) {
            const V2 t = o.dir * o.depth;
            const double x = pos.x + t.x, y = pos.y + t.y;
            X[l] = x;
            Y[l] = y;
            if (O.kind != 0) {
              if (O.kind == 1 && C.gain != 0.0) {
                const V2 lever = o.contact - V2{x, y};
                const double lever2 = norm2(lever);
                if (!(lever2 < 1e-12)) {
                  double dtheta = C.gain * cross(lever, t) / lever2;
                  dtheta = dclamp(dtheta, -0.2, 0.2);
                  const double th = wrap_angle(P.th(l) + dtheta);
                  double s, c;
                  glibc_sincos(th, &s, &c);
                  P.th(l) = th;
                  P.s(l) = s;
                  P.c(l) = c;
                }
              }
              lane_refresh(W, G, S, l, O.nv);
            }
            mp = o.depth;
          }
        }
      }
      __syncwarp();
      // pair broad phase (push_sim.cpp:107-108)
      unsigned cand[NW];
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        const double ex = X[pa[w]] - X[pb[w]], ey = Y[pa[w]] - Y[pb[w]];
        cand[w] = __ballot_sync(kFull, om[w] != 0u && !(ex * ex + ey * ey > rr2[w]));
      }
      // uniform lexicographic candidate sweep, narrow tests spread over lanes;
      // the word loop is not unrolled (the narrow-phase body is emitted once,
      // the per-word registers are picked by compare-select)
      int w = 0;
#pragma unroll 1
      while (w < NW) {
        unsigned cw = 0u;
#pragma unroll
        for (int v = 0; v < NW; ++v)
          if (v == w) cw = cand[v];
        if (!cw) {
          ++w;
          continue;
        }
        const int b = __ffs(cw) - 1;
#pragma unroll
        for (int v = 0; v < NW; ++v)
          if (v == w) cand[v] = cw & (cw - 1);
        const int p = 32 * w + b;
        const unsigned hm = warp_pair_poly(W, G, O, S, C, pij[p], l, &mp);
        if (hm) {
          // re-test the later active pairs touching i or j
#pragma unroll
          for (int v = 0; v < NW; ++v) {
            const bool touch = v >= w && (om[v] & hm) != 0u && 32 * v + l > p;
            const unsigned tm = __ballot_sync(kFull, touch);
            if (tm) {
              bool pass = false;
              if (touch) {
                const double fx = X[pa[v]] - X[pb[v]], fy = Y[pa[v]] - Y[pb[v]];
                pass = !(fx * fx + fy * fy > rr2[v]);
              }
              cand[v] = (cand[v] & ~tm) | __ballot_sync(kFull, pass);
            }
          }
        }
      }
      // clamp every object (push_sim.cpp:118 -> :48-54); a clamped polygon
      // moved, so its cached polygon is refreshed
      if (real) {
        double xo = X[l], yo = Y[l];
        bool moved = false;
        if (!(fabs(xo) <= hcl)) {
          X[l] = xo = fmin(fmax(xo, -hcl), hcl);
          moved = true;
        }
        if (!(fabs(yo) <= hcl)) {
          Y[l] = yo = fmin(fmax(yo, -hcl), hcl);
          moved = true;
        }
        if (moved && O.kind != 0) lane_refresh(W, G, S, l, O.nv);
      }
      if (!__any_sync(kFull, mp > C.eps_pen)) break;  // max_pen <= eps_pen
      // fixed point (see warp_resolve): every pose bit-identical to the
      // iteration start -> the remaining iterations of the substep repeat it
      const bool same = !real || (__double_as_longlong(X[l]) == __double_as_longlong(xs) &&
                                  __double_as_longlong(Y[l]) == __double_as_longlong(ys) &&
                                  __double_as_longlong(P.th(l)) == __double_as_longlong(ts));
      if (C.fixpoint && __all_sync(kFull, same)) break;
      __syncwarp();
    }
  }
  // final all-pairs check (world.cpp:139-152), order-free max
  __syncwarp();
  double worst = 0.0;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const int a = pa[w], b = pb[w];
    const int ka = __shfl_sync(kFull, O.kind, a), kb = __shfl_sync(kFull, O.kind, b);
    const int na = __shfl_sync(kFull, O.nv, a), nb = __shfl_sync(kFull, O.nv, b);
    const double ra = __shfl_sync(kFull, O.r, a), rb = __shfl_sync(kFull, O.r, b);
    const double fx = X[a] - X[b], fy = Y[a] - Y[b];
    if (32 * w + l < Pn && !(fx * fx + fy * fy > rr2[w]))
      worst = dmax(worst, lane_pair_depth(W, G, a, ka, na, ra, b, kb, nb, rb));
  }
  worst = warp_max(worst);
  *residual = worst;
  return worst > C.eps_pen ? 2 : 0;
}

}  // namespace

}  // namespace ppg
