// geom.cuh — FP64 2-D geometry for the device, operation-for-operation with
// the reference (arxiv 2207.06649 pushplan core; paths below are relative to
// /root/reference/proj/core).  Compiled with --fmad=false so every +,-,*
// rounds exactly like the reference's SSE2 code; / and sqrt are IEEE
// round-to-nearest on both sides.  std::max(a,b) == (a < b ? b : a),
// std::min(a,b) == (b < a ? b : a), std::clamp(v,lo,hi) ==
// (v < lo ? lo : hi < v ? hi : v): they decide signed zeros, which the FNV
// state digest (world.cpp:166-191) sees.
#pragma once

#include <cmath>
#include <cstdint>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

namespace ppg {

#ifdef __CUDACC__
#define PPG_DI __device__ __forceinline__
#define PPG_HD __host__ __device__ __forceinline__
#define PPG_ROLLED _Pragma("unroll 1")
#else
#define PPG_DI inline
#define PPG_HD inline
#define PPG_ROLLED
#endif

PPG_HD double inf_d() { return __builtin_huge_val(); }

struct V2 {
  double x, y;
};

PPG_HD V2 mk(double x, double y) { return V2{x, y}; }
PPG_HD V2 operator+(V2 a, V2 b) { return V2{a.x + b.x, a.y + b.y}; }  // geometry.hpp:12
PPG_HD V2 operator-(V2 a, V2 b) { return V2{a.x - b.x, a.y - b.y}; }  // geometry.hpp:13
PPG_HD V2 operator*(V2 a, double s) { return V2{a.x * s, a.y * s}; }  // geometry.hpp:14
PPG_HD V2 operator-(V2 a) { return V2{-a.x, -a.y}; }                  // geometry.hpp:15
PPG_HD double dot(V2 a, V2 b) { return a.x * b.x + a.y * b.y; }       // geometry.hpp:20
PPG_HD double cross(V2 a, V2 b) { return a.x * b.y - a.y * b.x; }     // geometry.hpp:21
PPG_HD double norm2(V2 a) { return a.x * a.x + a.y * a.y; }           // geometry.hpp:22
PPG_HD double norm(V2 a) { return sqrt(norm2(a)); }                   // geometry.hpp:23
PPG_HD V2 perp(V2 a) { return V2{-a.y, a.x}; }                        // geometry.hpp:24
PPG_HD V2 normalized(V2 a) {                                          // geometry.hpp:25-28
  const double n = norm(a);
  return n > 0.0 ? V2{a.x / n, a.y / n} : V2{0.0, 0.0};
}
PPG_HD double dmax(double a, double b) { return a < b ? b : a; }
PPG_HD double dmin(double a, double b) { return b < a ? b : a; }
PPG_HD double dclamp(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }

// geometry.cpp:8-13.  fmod is exact on both sides.
PPG_HD double wrap_angle(double theta) {
  const double two_pi = 2.0 * M_PI;
  double t = fmod(theta + M_PI, two_pi);
  if (t < 0.0) t += two_pi;
  return t - M_PI;
}

// geometry.cpp:15-22
PPG_HD V2 closest_point_on_segment(V2 p, V2 a, V2 b) {
  const V2 ab = b - a;
  const double len2 = norm2(ab);
  if (len2 == 0.0) return a;
  double t = dot(p - a, ab) / len2;
  t = dclamp(t, 0.0, 1.0);
  return a + ab * t;
}

// geometry.cpp:24-26
PPG_HD double dist_point_segment(V2 p, V2 a, V2 b) {
  return norm(p - closest_point_on_segment(p, a, b));
}

// geometry.cpp:28-40
PPG_HD double dist_segment_segment(V2 a0, V2 a1, V2 b0, V2 b1) {
  const double d1 = cross(a1 - a0, b0 - a0);
  const double d2 = cross(a1 - a0, b1 - a0);
  const double d3 = cross(b1 - b0, a0 - b0);
  const double d4 = cross(b1 - b0, a1 - b0);
  if (((d1 > 0) != (d2 > 0)) && ((d3 > 0) != (d4 > 0))) return 0.0;
  return dmin(dmin(dist_point_segment(b0, a0, a1), dist_point_segment(b1, a0, a1)),
              dmin(dist_point_segment(a0, b0, b1), dist_point_segment(a1, b0, b1)));
}

constexpr int kMaxV = 8;

// A convex polygon in world coordinates (reference Polygon, geometry.hpp:44).
struct Poly {
  int n;
  V2 p[kMaxV];
  PPG_HD V2 v(int i) const { return p[i]; }
};

// The same polygon held elsewhere: the per-warp shared-memory vertex cache of
// warp_poly.cuh.  The polygon functions below take either; their edge loops
// stay rolled (each unrolled copy carried a division, and the inlined copies
// made the polygon kernels overflow the instruction cache).
struct PolyRef {
  const V2* p;
  int n;
  PPG_HD V2 v(int i) const { return p[i]; }
};

// geometry.cpp:56-64
template <class PG>
PPG_HD bool point_in_convex(V2 p, const PG& poly) {
  PPG_ROLLED
  for (int i = 0; i < poly.n; ++i) {
    const V2 a = poly.v(i);
    const V2 b = poly.v(i + 1 == poly.n ? 0 : i + 1);
    if (cross(b - a, p - a) < 0.0) return false;
  }
  return true;
}

// geometry.cpp:66-79
template <class PG>
PPG_HD V2 polygon_centroid(const PG& poly) {
  double area2 = 0.0;
  V2 c{0.0, 0.0};
  PPG_ROLLED
  for (int i = 0; i < poly.n; ++i) {
    const V2 a = poly.v(i);
    const V2 b = poly.v(i + 1 == poly.n ? 0 : i + 1);
    const double w = cross(a, b);
    area2 += w;
    const V2 t = (a + b) * w;
    c.x += t.x;
    c.y += t.y;
  }
  if (area2 == 0.0) return poly.n == 0 ? V2{0.0, 0.0} : poly.v(0);
  return c * (1.0 / (3.0 * area2));
}

// geometry.cpp:81-85
PPG_HD double support_extent(const Poly& poly, V2 dir) {
  double best = -inf_d();
  for (int i = 0; i < poly.n; ++i) best = dmax(best, dot(poly.p[i], dir));
  return best;
}

// geometry.cpp:87-100
template <class PG>
PPG_HD V2 closest_point_on_polygon(V2 p, const PG& poly) {
  V2 best{0.0, 0.0};
  double best_d = inf_d();
  PPG_ROLLED
  for (int i = 0; i < poly.n; ++i) {
    const V2 q = closest_point_on_segment(p, poly.v(i), poly.v(i + 1 == poly.n ? 0 : i + 1));
    const double d = norm2(p - q);
    if (d < best_d) {
      best_d = d;
      best = q;
    }
  }
  return best;
}

// geometry.cpp:102-105
template <class PG>
PPG_HD double signed_dist_point_polygon(V2 p, const PG& poly) {
  const double d = norm(p - closest_point_on_polygon(p, poly));
  return point_in_convex(p, poly) ? -d : d;
}

struct Overlap {
  double depth;
  V2 dir;
  V2 contact;
};

// geometry.cpp:107-115
PPG_HD Overlap disc_disc_overlap(V2 ca, double ra, V2 cb, double rb) {
  Overlap o;
  const V2 d = cb - ca;
  const double dist = norm(d);
  o.depth = ra + rb - dist;
  o.dir = dist > 0.0 ? d * (1.0 / dist) : V2{1.0, 0.0};
  o.contact = ca + o.dir * ra;
  return o;
}

// geometry.cpp:117-132
template <class PG>
PPG_HD Overlap disc_polygon_overlap(V2 c, double r, const PG& poly) {
  Overlap o;
  const V2 q = closest_point_on_polygon(c, poly);
  const V2 d = q - c;
  const double dist = norm(d);
  o.contact = q;
  o.depth = point_in_convex(c, poly) ? r + dist : r - dist;
  o.dir = dist > 0.0 ? d * (1.0 / dist) : V2{1.0, 0.0};
  return o;
}

// geometry.cpp:137-152
PPG_HD bool sat_min_overlap(const Poly& a, const Poly& b, double& depth, V2& axis) {
  for (int i = 0; i < a.n; ++i) {
    const V2 edge = a.p[i + 1 == a.n ? 0 : i + 1] - a.p[i];
    const V2 normal = normalized(V2{edge.y, -edge.x});
    const double a_max = support_extent(a, normal);
    const double b_min = -support_extent(b, -normal);
    const double o = a_max - b_min;
    if (o < depth) {
      depth = o;
      axis = normal;
    }
    if (o <= 0.0) return false;
  }
  return true;
}

// geometry.cpp:191-195
PPG_HD bool polygons_intersect(const Poly& a, const Poly& b) {
  double depth = inf_d();
  V2 axis{0.0, 0.0};
  return sat_min_overlap(a, b, depth, axis) && sat_min_overlap(b, a, depth, axis);
}

// geometry.cpp:176-184
PPG_HD double dist_polygon_polygon(const Poly& a, const Poly& b) {
  if (polygons_intersect(a, b)) return 0.0;
  double best = inf_d();
  for (int i = 0; i < a.n; ++i)
    for (int j = 0; j < b.n; ++j)
      best = dmin(best, dist_segment_segment(a.p[i], a.p[i + 1 == a.n ? 0 : i + 1], b.p[j],
                                             b.p[j + 1 == b.n ? 0 : j + 1]));
  return best;
}

// geometry.cpp:156-174.  When the SAT finds a separating axis the reference
// returns depth = -dist_polygon_polygon(a, b) <= 0; every caller on the hot
// path (push_sim.cpp:96, :110; world.cpp:148 via max with 0.0) only tests
// depth > 0 or takes max(., 0.0) of it, so `exact_separation` = false skips
// that distance and returns depth = -0.0 (same decisions, same bits).
PPG_HD Overlap polygon_polygon_overlap(const Poly& a, const Poly& b, bool exact_separation) {
  Overlap o;
  o.contact = V2{0.0, 0.0};
  double depth = inf_d();
  V2 axis{0.0, 0.0};
  const bool ab = sat_min_overlap(a, b, depth, axis);
  const bool ba = ab && sat_min_overlap(b, a, depth, axis);
  if (!ab || !ba) {
    o.depth = exact_separation ? -dist_polygon_polygon(a, b) : -0.0;
    o.dir = normalized(polygon_centroid(b) - polygon_centroid(a));
    return o;
  }
  o.depth = depth;
  const V2 cb = polygon_centroid(b), ca = polygon_centroid(a);
  const V2 sep = cb - ca;
  o.dir = dot(sep, axis) >= 0.0 ? axis : -axis;
  o.contact = (closest_point_on_polygon(cb, a) + closest_point_on_polygon(ca, b)) * 0.5;
  return o;
}

}  // namespace ppg
