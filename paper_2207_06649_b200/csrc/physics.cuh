// physics.cuh — per-environment device functions of the hot path:
// resolve_push (push_sim.cpp:58-130), sample_pushes (actions.cpp:51-73),
// graspable (actions.cpp:113-147) and the keyed MT19937-64 stream
// (rng.hpp:8-23 + libstdc++ mersenne_twister_engine / uniform_int_distribution).
//
// Layout: one environment per lane.  Its poses live in shared memory as
// [x|y|theta][object] planes with a per-lane column (stride = threads per
// block), so a warp touching object i of 32 environments hits 32 consecutive
// 8-byte words (conflict-free).  Shapes are read from HBM in [object][table]
// SoA (table = env for per-env scenes -> coalesced; table 0 for a shared
// scene -> broadcast).
#pragma once

#include "geom.cuh"
#include "glibc_sincos.cuh"

namespace ppg {

constexpr int kMaxObjects = 32;
constexpr int kMaxNa = 32;        // pushes_per_object supported by the device sampler
constexpr int kGraspAngles = 16;  // actions.hpp:11
constexpr int kMaxGammaPow = 128;

// Per-launch constants, passed by value (__grid_constant__).  The angle
// tables are computed on the host with the same glibc cos/sin as the
// reference (actions.cpp:59-60, :77-78), as is gamma^k (mcts.cpp:132, :164).
struct SimConst {
  double tip_r, tip_clear;
  double push_distance;
  int substeps, max_iters;
  double eps_pen, gain;
  double side, margin;
  double finger_width, finger_thickness, opening, approach_clearance;
  double margin_threshold;
  int na;  // pushes_per_object
  int n;   // objects per environment
  int fixpoint;  // skip the rest of a substep at a bit-identical fixed point (PPG_NO_FIXPOINT=1: off)
  double dir_cos[kMaxNa], dir_sin[kMaxNa];
  double g_cos[kGraspAngles], g_sin[kGraspAngles];
  double gamma_pow[kMaxGammaPow];
};

struct ShapeView {
  const int* kind;      // [n][T]
  const double* rad;    // [n][T]
  const double* br;     // [n][T] bounding radius (world.cpp:32-37), precomputed
  const int* nv;        // [n][T]
  const double* verts;  // [T][n][kMaxV][2]
  int T;
  int t;  // this lane's table
  int n;
  PPG_DI int kind_(int i) const { return __ldg(kind + i * T + t); }
  PPG_DI double rad_(int i) const { return __ldg(rad + i * T + t); }
  PPG_DI double br_(int i) const { return __ldg(br + i * T + t); }
  PPG_DI int nv_(int i) const { return __ldg(nv + i * T + t); }
  PPG_DI V2 vert(int i, int k) const {
    const double* p = verts + ((static_cast<size_t>(t) * n + i) * kMaxV + k) * 2;
    return V2{__ldg(p), __ldg(p + 1)};
  }
};

// Planes x | y | theta | cos(theta) | sin(theta) (the last two cached for
// polygons: world_polygon is a pure function of the pose, so computing the
// glibc sincos once per rotation instead of in every narrow test is exact).
struct PoseView {
  double* p;
  int stride;
  int n;
  PPG_DI double& x(int i) const { return p[i * stride]; }
  PPG_DI double& y(int i) const { return p[(n + i) * stride]; }
  PPG_DI double& th(int i) const { return p[(2 * n + i) * stride]; }
  PPG_DI double& c(int i) const { return p[(3 * n + i) * stride]; }
  PPG_DI double& s(int i) const { return p[(4 * n + i) * stride]; }
  PPG_DI V2 pos(int i) const { return V2{x(i), y(i)}; }
};
constexpr int kPosePlanes = 5;

// Refreshes the cached rotation of polygon i (after its theta changed).
PPG_DI void refresh_trig(const PoseView& P, int i) {
  double s, c;
  glibc_sincos(P.th(i), &s, &c);  // bit-identical to the reference's libm sincos
  P.s(i) = s;
  P.c(i) = c;
}

PPG_DI void refresh_all_trig(const PoseView& P, const ShapeView& S) {
  for (int i = 0; i < P.n; ++i)
    if (S.kind_(i) != 0) refresh_trig(P, i);
}

// world.cpp:57-62 (Vec2::rotated geometry.hpp:29-32), with the rotation's
// sincos from the cache.
PPG_DI void world_polygon(const PoseView& P, const ShapeView& S, int i, Poly& out) {
  const double s = P.s(i), c = P.c(i);
  const V2 pos = P.pos(i);
  out.n = S.nv_(i);
  for (int k = 0; k < out.n; ++k) {
    const V2 v = S.vert(i, k);
    out.p[k] = pos + V2{c * v.x - s * v.y, s * v.x + c * v.y};
  }
}

// world.cpp:101-107
PPG_DI double object_point_distance(const PoseView& P, const ShapeView& S, int i, V2 p) {
  if (S.kind_(i) == 0) return dmax(0.0, norm(p - P.pos(i)) - S.rad_(i));
  Poly poly;
  world_polygon(P, S, i, poly);
  return dmax(0.0, signed_dist_point_polygon(p, poly));
}

// world.cpp:154-164
PPG_DI bool collides_gripper_start(const PoseView& P, const ShapeView& S, const SimConst& C, V2 p) {
  const double r = C.tip_r + C.tip_clear;
  const double h = C.side / 2.0;
  if (p.x - r < -h || p.x + r > h || p.y - r < -h || p.y + r > h) return true;
  for (int i = 0; i < S.n; ++i) {
    if (S.kind_(i) == 0) {
      // a disc farther than (r + radius)(1 + 1e-12) cannot pass the exact
      // test (norm and the subtraction round by < 1e-15 relative): skip its
      // square root; the rest take the reference's expression
      const V2 dv = p - P.pos(i);
      const double lim = r + S.rad_(i);
      if (dv.x * dv.x + dv.y * dv.y > lim * lim * (1.0 + 1e-12)) continue;
    }
    if (object_point_distance(P, S, i, p) < r) return true;
  }
  return false;
}

// push_sim.cpp:20-32 (== world.cpp:123-135)
PPG_DI Overlap object_pair_overlap(const PoseView& P, const ShapeView& S, int a, int b) {
  const bool da = S.kind_(a) == 0, db = S.kind_(b) == 0;
  if (da && db) return disc_disc_overlap(P.pos(a), S.rad_(a), P.pos(b), S.rad_(b));
  Poly pa, pb;
  if (da) {
    world_polygon(P, S, b, pb);
    return disc_polygon_overlap(P.pos(a), S.rad_(a), pb);
  }
  if (db) {
    world_polygon(P, S, a, pa);
    Overlap o = disc_polygon_overlap(P.pos(b), S.rad_(b), pa);
    o.dir = -o.dir;
    return o;
  }
  world_polygon(P, S, a, pa);
  world_polygon(P, S, b, pb);
  return polygon_polygon_overlap(pa, pb, false);
}

// push_sim.cpp:13-18
PPG_DI Overlap tip_object_overlap(const PoseView& P, const ShapeView& S, V2 tc, double tr, int i) {
  if (S.kind_(i) == 0) return disc_disc_overlap(tc, tr, P.pos(i), S.rad_(i));
  Poly poly;
  world_polygon(P, S, i, poly);
  return disc_polygon_overlap(tc, tr, poly);
}

// push_sim.cpp:36-46
PPG_DI void apply_contact_motion(const PoseView& P, const ShapeView& S, int i, V2 t, V2 contact,
                                 double gain) {
  P.x(i) += t.x;
  P.y(i) += t.y;
  if (S.kind_(i) != 1 || gain == 0.0) return;
  const V2 lever = contact - P.pos(i);
  const double lever2 = norm2(lever);
  if (lever2 < 1e-12) return;
  double dtheta = gain * cross(lever, t) / lever2;
  dtheta = dclamp(dtheta, -0.2, 0.2);
  P.th(i) = wrap_angle(P.th(i) + dtheta);
  refresh_trig(P, i);
}

// world.cpp:139-152
template <bool kCount>
PPG_DI double max_pairwise_penetration(const PoseView& P, const ShapeView& S, long long* pfinal) {
  double worst = 0.0;
  for (int i = 0; i + 1 < S.n; ++i)
    for (int j = i + 1; j < S.n; ++j) {
      const double reach = S.br_(i) + S.br_(j);
      if (norm2(P.pos(i) - P.pos(j)) > reach * reach) continue;
      if (kCount) ++*pfinal;
      worst = dmax(worst, object_pair_overlap(P, S, i, j).depth);
    }
  return worst;
}

struct Counts {
  long long tb, tn, ht, pb, pn, hp, s, pfinal;
};

// resolve_push (push_sim.cpp:58-130).  Returns 0 ok, 1 start collision,
// 2 not converged; *residual = final max pairwise penetration.  check_start
// = false only where the push came from sample_pushes on this same state,
// which already evaluated the identical collides_gripper_start test
// (actions.cpp:68) — the result is then known to be false.
template <bool kCount>
PPG_DI int resolve_push(const PoseView& P, const ShapeView& S, const SimConst& C, V2 start, V2 end,
                        bool check_start, double* residual, Counts* cnt) {
  if (check_start && collides_gripper_start(P, S, C, start)) return 1;
  const int n = S.n;
  const V2 delta = (end - start) * (1.0 / C.substeps);
  const double sweep_reach = C.push_distance + C.tip_r;
  uint32_t active = 0;
  {
    double max_diam = 0.0;
    for (int i = 0; i < n; ++i) max_diam = dmax(max_diam, 2.0 * S.br_(i));
    const double reach = sweep_reach + 2.0 * max_diam;
    for (int i = 0; i < n; ++i) {
      const double d = dist_point_segment(P.pos(i), start, end);
      if (d <= reach + S.br_(i)) active |= 1u << i;
    }
  }
  const double h = C.side / 2.0 - C.margin - 1e-9;  // clamp_to_boundary push_sim.cpp:48-54
  for (int step = 1; step <= C.substeps; ++step) {
    const V2 tc = start + delta * static_cast<double>(step);
    if (kCount) cnt->s++;
    for (int iter = 0; iter < C.max_iters; ++iter) {
      double max_pen = 0.0;
      // fixed-point check (not in the work-counting variant, which must count
      // every reference iteration): iteration-start poses of a long substep
      double sx[kMaxObjects], sy[kMaxObjects], st[kMaxObjects];
      const bool fixcheck = !kCount && C.fixpoint && iter >= 6;
      if (fixcheck)
        for (int i = 0; i < n; ++i) {
          sx[i] = P.x(i);
          sy[i] = P.y(i);
          st[i] = P.th(i);
        }
      for (int i = 0; i < n; ++i) {
        if (!(active >> i & 1u)) continue;
        const double reach = C.tip_r + S.br_(i);
        if (kCount) cnt->tb++;
        if (norm2(P.pos(i) - tc) > reach * reach) continue;
        if (kCount) cnt->tn++;
        const Overlap o = tip_object_overlap(P, S, tc, C.tip_r, i);
        if (o.depth > 0.0) {
          if (kCount) cnt->ht++;
          apply_contact_motion(P, S, i, o.dir * o.depth, o.contact, C.gain);
          max_pen = dmax(max_pen, o.depth);
        }
      }
      for (int i = 0; i + 1 < n; ++i) {
        if (!(active >> i & 1u)) continue;
        const double bri = S.br_(i);
        for (int j = i + 1; j < n; ++j) {
          if (!(active >> j & 1u)) continue;
          const double reach = bri + S.br_(j);
          if (kCount) cnt->pb++;
          if (norm2(P.pos(i) - P.pos(j)) > reach * reach) continue;
          if (kCount) cnt->pn++;
          const Overlap o = object_pair_overlap(P, S, i, j);
          if (o.depth > 0.0) {
            if (kCount) cnt->hp++;
            apply_contact_motion(P, S, i, -o.dir * (0.5 * o.depth), o.contact, C.gain);
            apply_contact_motion(P, S, j, o.dir * (0.5 * o.depth), o.contact, C.gain);
            max_pen = dmax(max_pen, o.depth);
          }
        }
      }
      for (int i = 0; i < n; ++i) {
        P.x(i) = dclamp(P.x(i), -h, h);
        P.y(i) = dclamp(P.y(i), -h, h);
      }
      if (max_pen <= C.eps_pen) break;
      if (fixcheck) {  // every pose bit-identical: the rest of the substep repeats this iteration
        bool same = true;
        for (int i = 0; i < n; ++i)
          same = same && __double_as_longlong(P.x(i)) == __double_as_longlong(sx[i]) &&
                 __double_as_longlong(P.y(i)) == __double_as_longlong(sy[i]) &&
                 __double_as_longlong(P.th(i)) == __double_as_longlong(st[i]);
        if (same) break;
      }
    }
  }
  const double final_pen = max_pairwise_penetration<kCount>(P, S, kCount ? &cnt->pfinal : nullptr);
  if (residual) *residual = final_pen;
  return final_pen > C.eps_pen ? 2 : 0;
}

// actions.cpp:12-30
PPG_DI double contour_radius(const PoseView& P, const ShapeView& S, int i, V2 d) {
  if (S.kind_(i) == 0) return S.rad_(i);
  double s, c;
  glibc_sincos(-P.th(i), &s, &c);
  const V2 dl{c * d.x - s * d.y, s * d.x + c * d.y};
  double best = 0.0;
  const int nv = S.nv_(i);
  for (int k = 0; k < nv; ++k) {
    const V2 a = S.vert(i, k);
    const V2 b = S.vert(i, k + 1 == nv ? 0 : k + 1);
    const V2 e = b - a;
    const double denom = cross(dl, e);
    if (fabs(denom) < 1e-15) continue;
    const double t = cross(a, e) / denom;
    const double sp = cross(a, dl) / denom;
    if (t > 0.0 && sp >= -1e-12 && sp <= 1.0 + 1e-12) best = dmax(best, t);
  }
  return best;
}

// Candidate (object o, angle k) of sample_pushes (actions.cpp:55-70).
// Returns false when the candidate is skipped; start/end are written when
// the geometric tests pass.  `full` also runs the start-collision filter.
PPG_DI bool push_candidate(const PoseView& P, const ShapeView& S, const SimConst& C, int o, int k,
                           bool full, V2& start, V2& end) {
  const V2 center = P.pos(o);
  const V2 d{C.dir_cos[k], C.dir_sin[k]};
  const double cr = contour_radius(P, S, o, d);
  if (cr <= 0.0) return false;
  const double offset = C.tip_r + C.tip_clear + 1e-9;
  start = center + d * (cr + offset);
  const V2 dir = normalized(center - start);
  end = start + dir * C.push_distance;
  // push_action_valid world.cpp:86-90 with Workspace::contains_point world.hpp:23-26
  const double len = norm(end - start);
  if (fabs(len - C.push_distance) > 1e-9) return false;
  const double hh = C.side / 2.0;
  if (!(start.x > -hh && start.x < hh && start.y > -hh && start.y < hh)) return false;
  if (!(end.x > -hh && end.x < hh && end.y > -hh && end.y < hh)) return false;
  if (full && collides_gripper_start(P, S, C, start)) return false;
  return true;
}

// actions.cpp:32-39
PPG_DI double rect_min_wall_clearance(const Poly& rect, double side) {
  const double h = side / 2.0;
  double best = inf_d();
  for (int i = 0; i < rect.n; ++i)
    best = dmin(best, dmin(h - fabs(rect.p[i].x), h - fabs(rect.p[i].y)));
  return best;
}

// actions.cpp:41-47
PPG_DI double rect_object_distance(const Poly& rect, const PoseView& P, const ShapeView& S, int i) {
  if (S.kind_(i) == 0) {
    const double sd = signed_dist_point_polygon(P.pos(i), rect);
    return dmax(0.0, sd - S.rad_(i));
  }
  Poly poly;
  world_polygon(P, S, i, poly);
  return dist_polygon_polygon(rect, poly);
}

struct GraspOut {
  bool graspable;
  double margin;
  double x, y;
  int k;  // -1: no feasible pose
};

// One grasp angle k of graspable (actions.cpp:118-140) with grasp_fingers
// (actions.cpp:75-111).  Returns true when the pose is feasible; *margin is
// its minimum obstacle clearance and (cx, cy) the grasp centre.
PPG_DI bool grasp_angle(const PoseView& P, const ShapeView& S, const SimConst& C, int target, int k,
                        double* margin_out, double* cx, double* cy) {
  const double ht = C.finger_thickness / 2.0;
  const double hw = C.finger_width / 2.0;
  const V2 u{C.g_cos[k], C.g_sin[k]};
  const V2 v = perp(u);
  double lo_u, hi_u, lo_v, hi_v;
  if (S.kind_(target) == 0) {
    const V2 tp = P.pos(target);
    const double r = S.rad_(target);
    const double cu = dot(tp, u);
    const double cv = dot(tp, v);
    lo_u = cu - r;
    hi_u = cu + r;
    lo_v = cv - r;
    hi_v = cv + r;
  } else {
    Poly tpoly;
    world_polygon(P, S, target, tpoly);
    hi_u = support_extent(tpoly, u);
    lo_u = -support_extent(tpoly, -u);
    hi_v = support_extent(tpoly, v);
    lo_v = -support_extent(tpoly, -v);
  }
  const double extent = hi_u - lo_u;
  if (!(extent < C.opening - 2.0 * C.approach_clearance)) return false;
  const V2 center = u * ((lo_u + hi_u) / 2.0) + v * ((lo_v + hi_v) / 2.0);
  Poly ra, rb;
  {
    const V2 ca = center + u * (-(C.opening / 2.0 + ht));
    const V2 cb = center + u * (C.opening / 2.0 + ht);
    ra.n = rb.n = 4;
    ra.p[0] = ca - u * ht - v * hw;
    ra.p[1] = ca + u * ht - v * hw;
    ra.p[2] = ca + u * ht + v * hw;
    ra.p[3] = ca - u * ht + v * hw;
    rb.p[0] = cb - u * ht - v * hw;
    rb.p[1] = cb + u * ht - v * hw;
    rb.p[2] = cb + u * ht + v * hw;
    rb.p[3] = cb - u * ht + v * hw;
  }
  if (dmin(rect_min_wall_clearance(ra, C.side), rect_min_wall_clearance(rb, C.side)) <= 0.0) return false;
  double margin = C.side;
  for (int i = 0; i < S.n; ++i) {
    if (i == target) continue;
    const double d = dmin(rect_object_distance(ra, P, S, i), rect_object_distance(rb, P, S, i));
    if (d <= 0.0) return false;
    margin = dmin(margin, d);
  }
  *margin_out = margin;
  *cx = center.x;
  *cy = center.y;
  return true;
}

// graspable (actions.cpp:113-147): first strict maximum of the margin over
// feasible angles in index order.
PPG_DI GraspOut graspable(const PoseView& P, const ShapeView& S, const SimConst& C, int target) {
  double best_margin = -1.0;
  GraspOut g{false, 0.0, 0.0, 0.0, -1};
  for (int k = 0; k < kGraspAngles; ++k) {
    double margin, cx, cy;
    if (grasp_angle(P, S, C, target, k, &margin, &cx, &cy) && margin > best_margin) {
      best_margin = margin;
      g.k = k;
      g.x = cx;
      g.y = cy;
    }
  }
  if (g.k >= 0) {
    g.margin = best_margin;
    g.graspable = best_margin >= C.margin_threshold;
  }
  return g;
}

// ---------------- keyed RNG ----------------

PPG_DI uint64_t splitmix64(uint64_t x) {  // rng.hpp:8-13
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
PPG_DI uint64_t mix_keys(uint64_t seed, uint64_t a, uint64_t b) {  // rng.hpp:15-17
  return splitmix64(splitmix64(splitmix64(seed) ^ a) ^ b);
}

// std::mt19937_64 with its 312-word state in HBM, word-major [312][E] so a
// warp's accesses to word w of 32 environments coalesce.  Seeding and the
// block twist follow libstdc++ random.tcc (seed(), _M_gen_rand()).
struct MtView {
  uint64_t* mt;  // &state[0][e]
  int stride;    // E
  bool frozen = false;  // speculative use: a draw that needs a twist aborts (idx = kMtFrozen)
  PPG_DI uint64_t& w(int i) const { return mt[static_cast<size_t>(i) * stride]; }
};

PPG_DI void mt_seed(const MtView& g, uint64_t seed) {
  uint64_t prev = seed;
  g.w(0) = seed;
  for (int i = 1; i < 312; ++i) {
    prev = 6364136223846793005ull * (prev ^ (prev >> 62)) + static_cast<uint64_t>(i);
    g.w(i) = prev;
  }
}

PPG_DI uint64_t mt_next(const MtView& g, int& idx) {
  const uint64_t UM = 0xffffffff80000000ull, LM = 0x7fffffffull, A = 0xb5026f5aa96619e9ull;
  if (idx >= 312) {
    uint64_t cur = g.w(0);
    for (int k = 0; k < 311; ++k) {
      const uint64_t nxt = g.w(k + 1);
      const uint64_t y = (cur & UM) | (nxt & LM);
      const uint64_t far = k < 156 ? g.w(k + 156) : g.w(k - 156);
      g.w(k) = far ^ (y >> 1) ^ ((y & 1) ? A : 0);
      cur = nxt;
    }
    const uint64_t y = (cur & UM) | (g.w(0) & LM);
    g.w(311) = g.w(155) ^ (y >> 1) ^ ((y & 1) ? A : 0);
    idx = 0;
  }
  uint64_t z = g.w(idx++);
  z ^= (z >> 29) & 0x5555555555555555ull;
  z ^= (z << 17) & 0x71d67fffeda60000ull;
  z ^= (z << 37) & 0xfff7eee000000000ull;
  z ^= (z >> 43);
  return z;
}

// uniform_int_distribution<size_t>(0, n-1)(mt19937_64): Lemire _S_nd with a
// 128-bit product (uniform_int_dist.h:255-280, 313-321).
PPG_DI uint64_t mt_pick(const MtView& g, int& idx, uint64_t n) {
  uint64_t x = mt_next(g, idx);
  uint64_t low = x * n;
  uint64_t high = __umul64hi(x, n);
  if (low < n) {
    const uint64_t thr = (0ull - n) % n;
    while (low < thr) {
      x = mt_next(g, idx);
      low = x * n;
      high = __umul64hi(x, n);
    }
  }
  return high;
}

}  // namespace ppg
