// host_scenes.cpp — host-side input generators that feed the hot path:
// the synthetic clutter scenes of the reference harness (bench::generate_case
// / generate_case_motif, bench.cpp:234-317) and the keyed uniform picks of
// rng.hpp:21-23 + mcts.cpp:151-152.  They use the same libstdc++
// std::mt19937_64 / uniform_*_distribution and glibc cos/sin as the
// reference, and the shared FP64 geometry of geom.cuh (host path), so the
// generated scenes are bit-identical to the reference's (checked by
// tests/test_scenes.py against oracle/_ref).  Threads split the seeds.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

#include "geom.cuh"
#include "pushplan_gpu.h"

namespace {

using ppg::V2;

uint64_t splitmix64(uint64_t x) {  // rng.hpp:8-13
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
uint64_t mix_keys(uint64_t seed, uint64_t a, uint64_t b) {  // rng.hpp:15-17
  return splitmix64(splitmix64(splitmix64(seed) ^ a) ^ b);
}

struct Obj {
  int kind = 0;  // 0 disc, 1 polygon
  double r = 0.0;
  int nv = 0;
  V2 v[ppg::kMaxV];
  double x = 0.0, y = 0.0, th = 0.0;
  double br() const {  // world.cpp:32-37
    if (kind == 0) return r;
    double best = 0.0;
    for (int k = 0; k < nv; ++k) best = std::max(best, ppg::norm(v[k]));
    return best;
  }
  ppg::Poly world() const {  // world.cpp:57-62
    ppg::Poly p;
    p.n = nv;
    for (int k = 0; k < nv; ++k) {
      const double c = std::cos(th), s = std::sin(th);
      p.p[k] = V2{x, y} + V2{c * v[k].x - s * v[k].y, s * v[k].x + c * v[k].y};
    }
    return p;
  }
};

double uniform(std::mt19937_64& rng, double lo, double hi) {  // bench.cpp:197-199
  return std::uniform_real_distribution<double>(lo, hi)(rng);
}

// geometry.cpp:42-54
bool is_ccw_convex(const ppg::Poly& poly) {
  const int n = poly.n;
  if (n < 3) return false;
  double area2 = 0.0;
  for (int i = 0; i < n; ++i) {
    const V2 a = poly.p[i], b = poly.p[(i + 1) % n], c = poly.p[(i + 2) % n];
    if (ppg::cross(b - a, c - b) <= 0.0) return false;
    area2 += ppg::cross(a, b);
  }
  return area2 > 0.0;
}

// bench.cpp:201-219 (ObjectShape::validate world.cpp:39-50 for the polygon)
Obj random_shape(std::mt19937_64& rng, double polygon_fraction) {
  Obj o;
  const double r = uniform(rng, 0.013, 0.021);
  if (uniform(rng, 0.0, 1.0) >= polygon_fraction) {
    o.kind = 0;
    o.r = r;
    return o;
  }
  const int sides = std::uniform_int_distribution<int>(5, 7)(rng);
  ppg::Poly poly;
  poly.n = sides;
  for (int i = 0; i < sides; ++i) {
    const double a = 2.0 * M_PI * i / sides + uniform(rng, -0.1, 0.1);
    const double rr = r * uniform(rng, 0.85, 1.0);
    poly.p[i] = V2{rr * std::cos(a), rr * std::sin(a)};
  }
  bool ok = is_ccw_convex(poly) && ppg::point_in_convex(V2{0.0, 0.0}, poly);
  for (int i = 0; i < sides && ok; ++i) ok = std::isfinite(poly.p[i].x) && std::isfinite(poly.p[i].y);
  if (!ok) {
    o.kind = 0;
    o.r = r;
    return o;
  }
  o.kind = 1;
  o.nv = sides;
  for (int i = 0; i < sides; ++i) o.v[i] = poly.p[i];
  return o;
}

// world.cpp:109-119 with dist_disc_polygon geometry.cpp:186-189
double object_object_distance(const Obj& a, const Obj& b) {
  const bool da = a.kind == 0, db = b.kind == 0;
  if (da && db) return std::max(0.0, ppg::norm(V2{a.x, a.y} - V2{b.x, b.y}) - a.r - b.r);
  if (da) return std::max(0.0, ppg::signed_dist_point_polygon(V2{a.x, a.y}, b.world()) - a.r);
  if (db) return std::max(0.0, ppg::signed_dist_point_polygon(V2{b.x, b.y}, a.world()) - b.r);
  return ppg::dist_polygon_polygon(a.world(), b.world());
}

// bench.cpp:221-230
bool placeable(const std::vector<Obj>& objs, const Obj& c, double gap) {
  const double h = 0.288 / 2.0;
  const double br = c.br();
  if (std::abs(c.x) + br > h - 0.004 || std::abs(c.y) + br > h - 0.004) return false;
  for (const Obj& o : objs)
    if (object_object_distance(c, o) < gap) return false;
  return true;
}

// world.cpp:123-152 on the generated scene (validate() penetration bound).
double max_penetration(const std::vector<Obj>& objs) {
  double worst = 0.0;
  for (size_t i = 0; i + 1 < objs.size(); ++i)
    for (size_t j = i + 1; j < objs.size(); ++j) {
      const Obj& a = objs[i];
      const Obj& b = objs[j];
      const double reach = a.br() + b.br();
      if (ppg::norm2(V2{a.x, a.y} - V2{b.x, b.y}) > reach * reach) continue;
      double depth;
      if (a.kind == 0 && b.kind == 0) depth = ppg::disc_disc_overlap(V2{a.x, a.y}, a.r, V2{b.x, b.y}, b.r).depth;
      else if (a.kind == 0) depth = ppg::disc_polygon_overlap(V2{a.x, a.y}, a.r, b.world()).depth;
      else if (b.kind == 0) depth = ppg::disc_polygon_overlap(V2{b.x, b.y}, b.r, a.world()).depth;
      else depth = ppg::polygon_polygon_overlap(a.world(), b.world(), false).depth;
      worst = std::max(worst, depth);
    }
  return worst;
}

// bench.cpp:234-317.  Returns false on rejection-sampling exhaustion
// (BenchError) or a scene that fails WorldState::validate.
bool generate(int motif, int n_objects, double pf, uint64_t seed, std::vector<Obj>& objs) {
  objs.clear();
  if (n_objects < 1) return false;
  if (motif == 0) {
    std::mt19937_64 rng(mix_keys(seed, 0xCA5E, 0));
    Obj target = random_shape(rng, pf);
    target.x = uniform(rng, -0.01, 0.01);
    target.y = uniform(rng, -0.01, 0.01);
    target.th = 0.0;
    objs.push_back(target);
    int attempts = 0;
    while (static_cast<int>(objs.size()) < n_objects) {
      if (++attempts > 10000) return false;
      Obj o = random_shape(rng, pf);
      const double radius = std::abs(uniform(rng, 0.0, 0.055)) + 0.03;
      const double angle = uniform(rng, -M_PI, M_PI);
      o.x = radius * std::cos(angle);
      o.y = radius * std::sin(angle);
      o.th = ppg::wrap_angle(uniform(rng, -M_PI, M_PI));
      if (!placeable(objs, o, 0.0015)) continue;
      objs.push_back(o);
    }
  } else {
    std::mt19937_64 rng(mix_keys(seed, 0x30F1F, 0));
    Obj target;
    target.kind = 0;
    target.r = uniform(rng, 0.014, 0.018);
    if (motif == 1) {
      target.x = uniform(rng, -0.008, 0.008);
      target.y = uniform(rng, -0.008, 0.008);
      objs.push_back(target);
      const int ring = std::min(n_objects - 1, 6);
      const double phase = uniform(rng, -M_PI, M_PI);
      for (int i = 0; i < ring; ++i) {
        Obj o;
        o.r = uniform(rng, 0.014, 0.019);
        const double a = phase + 2.0 * M_PI * i / ring + uniform(rng, -0.06, 0.06);
        const double d = target.r + o.r + uniform(rng, 0.002, 0.005);
        o.x = target.x + d * std::cos(a);
        o.y = target.y + d * std::sin(a);
        if (placeable(objs, o, 0.0012)) objs.push_back(o);
      }
    } else {
      const double h = 0.144;
      target.x = uniform(rng, -0.02, 0.02);
      target.y = -(h - target.r - 0.012);
      objs.push_back(target);
      const int wall = std::min(n_objects - 1, 5);
      for (int i = 0; i < wall; ++i) {
        Obj o;
        o.r = uniform(rng, 0.015, 0.02);
        const double x = target.x + (i - (wall - 1) / 2.0) * 0.037 + uniform(rng, -0.002, 0.002);
        const double y = target.y + target.r + o.r + uniform(rng, 0.0015, 0.004);
        o.x = x;
        o.y = y;
        if (placeable(objs, o, 0.0012)) objs.push_back(o);
      }
    }
    int attempts = 0;
    while (static_cast<int>(objs.size()) < n_objects) {
      if (++attempts > 10000) return false;
      Obj o = random_shape(rng, pf);
      const double radius = uniform(rng, 0.06, 0.11);
      const double angle = uniform(rng, -M_PI, M_PI);
      o.x = radius * std::cos(angle);
      o.y = radius * std::sin(angle);
      o.th = ppg::wrap_angle(uniform(rng, -M_PI, M_PI));
      if (!placeable(objs, o, 0.003)) continue;
      objs.push_back(o);
    }
  }
  const double h = 0.144;
  for (const Obj& o : objs)
    if (!(std::abs(o.x) < h && std::abs(o.y) < h)) return false;
  return max_penetration(objs) <= 1e-4;
}

}  // namespace

extern "C" {

int ppg_generate_cases(int motif, int n_objects, double polygon_fraction, const uint64_t* seeds, int count,
                       int32_t* kind, double* radius, int32_t* n_vertices, double* vertices, double* poses,
                       int32_t* target_index, int32_t* ok, int threads) {
  if (n_objects < 1 || n_objects > PPG_MAX_OBJECTS || count < 0 || motif < 0 || motif > 2) return PPG_EINVAL;
  const int n = n_objects;
  auto work = [&](int lo, int hi) {
    std::vector<Obj> objs;
    for (int c = lo; c < hi; ++c) {
      const bool good = generate(motif, n, polygon_fraction, seeds[c], objs);
      ok[c] = good ? 1 : 0;
      target_index[c] = 0;
      for (int i = 0; i < n; ++i) {
        const Obj o = good ? objs[i] : Obj{};
        const size_t s = static_cast<size_t>(c) * n + i;
        kind[s] = o.kind;
        radius[s] = o.kind == 0 ? o.r : 0.0;
        n_vertices[s] = o.nv;
        for (int k = 0; k < PPG_MAX_VERTICES; ++k) {
          vertices[(s * PPG_MAX_VERTICES + k) * 2] = k < o.nv ? o.v[k].x : 0.0;
          vertices[(s * PPG_MAX_VERTICES + k) * 2 + 1] = k < o.nv ? o.v[k].y : 0.0;
        }
        poses[s * 3] = o.x;
        poses[s * 3 + 1] = o.y;
        poses[s * 3 + 2] = o.th;
      }
    }
  };
  const int t = std::max(1, std::min(threads, count / 64 + 1));
  std::vector<std::thread> pool;
  for (int k = 0; k < t; ++k) pool.emplace_back(work, count * k / t, count * (k + 1) / t);
  for (auto& th : pool) th.join();
  return PPG_SUCCESS;
}

int ppg_keyed_picks(uint64_t seed, const uint64_t* a, const uint64_t* b, const uint64_t* n, int count,
                    uint64_t* out) {
  for (int c = 0; c < count; ++c) {
    if (n[c] == 0) {
      out[c] = 0;
      continue;
    }
    std::mt19937_64 rng(mix_keys(seed, a ? a[c] : 0, b ? b[c] : 0));
    out[c] = std::uniform_int_distribution<size_t>(0, n[c] - 1)(rng);
  }
  return PPG_SUCCESS;
}

}  // extern "C"
