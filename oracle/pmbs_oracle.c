/*
 * pmbs_oracle.c — TEST INFRASTRUCTURE ONLY (see pmbs_oracle.h).
 *
 * Plain-C restatement of the reference's hot path, operation for operation,
 * so IEEE double results are bit-identical to the reference built with its
 * Release flags (no FMA contraction: compiled -ffp-contract=off).  Every
 * function cites the reference file:line it restates (paths relative to
 * /root/reference/proj/core).  std::max(a,b) is restated as (a < b ? b : a),
 * std::min(a,b) as (b < a ? b : a) and std::clamp(v,lo,hi) as
 * (v < lo ? lo : hi < v ? hi : v) — these decide signed zeros, which the
 * FNV state digest sees.
 */
#define _GNU_SOURCE
#include "pmbs_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef struct { double x, y; } v2;

static inline v2 V(double x, double y) { v2 r = {x, y}; return r; }
static inline v2 add(v2 a, v2 b) { return V(a.x + b.x, a.y + b.y); }        /* geometry.hpp:12 */
static inline v2 sub(v2 a, v2 b) { return V(a.x - b.x, a.y - b.y); }        /* geometry.hpp:13 */
static inline v2 mul(v2 a, double s) { return V(a.x * s, a.y * s); }        /* geometry.hpp:14 */
static inline v2 neg(v2 a) { return V(-a.x, -a.y); }                        /* geometry.hpp:15 */
static inline double dot(v2 a, v2 b) { return a.x * b.x + a.y * b.y; }      /* geometry.hpp:20 */
static inline double cross(v2 a, v2 b) { return a.x * b.y - a.y * b.x; }    /* geometry.hpp:21 */
static inline double norm2(v2 a) { return a.x * a.x + a.y * a.y; }          /* geometry.hpp:22 */
static inline double norm(v2 a) { return sqrt(norm2(a)); }                  /* geometry.hpp:23 */
static inline v2 perp(v2 a) { return V(-a.y, a.x); }                        /* geometry.hpp:24 */
static inline v2 normalized(v2 a) {                                         /* geometry.hpp:25-28 */
  const double n = norm(a);
  return n > 0.0 ? V(a.x / n, a.y / n) : V(0.0, 0.0);
}
static inline v2 rotated(v2 a, double th) {                                 /* geometry.hpp:29-32 */
  const double c = cos(th), s = sin(th);
  return V(c * a.x - s * a.y, s * a.x + c * a.y);
}
static inline double dmax(double a, double b) { return a < b ? b : a; }
static inline double dmin(double a, double b) { return b < a ? b : a; }
static inline double dclamp(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }

/* geometry.cpp:8-13 */
static double wrap_angle(double theta) {
  const double two_pi = 2.0 * M_PI;
  double t = fmod(theta + M_PI, two_pi);
  if (t < 0.0) t += two_pi;
  return t - M_PI;
}

/* geometry.cpp:15-22 */
static v2 closest_point_on_segment(v2 p, v2 a, v2 b) {
  const v2 ab = sub(b, a);
  const double len2 = norm2(ab);
  if (len2 == 0.0) return a;
  double t = dot(sub(p, a), ab) / len2;
  t = dclamp(t, 0.0, 1.0);
  return add(a, mul(ab, t));
}

/* geometry.cpp:24-26 */
static double dist_point_segment(v2 p, v2 a, v2 b) { return norm(sub(p, closest_point_on_segment(p, a, b))); }

/* geometry.cpp:28-40 */
static double dist_segment_segment(v2 a0, v2 a1, v2 b0, v2 b1) {
  const double d1 = cross(sub(a1, a0), sub(b0, a0));
  const double d2 = cross(sub(a1, a0), sub(b1, a0));
  const double d3 = cross(sub(b1, b0), sub(a0, b0));
  const double d4 = cross(sub(b1, b0), sub(a1, b0));
  if (((d1 > 0) != (d2 > 0)) && ((d3 > 0) != (d4 > 0))) return 0.0;
  return dmin(dmin(dist_point_segment(b0, a0, a1), dist_point_segment(b1, a0, a1)),
              dmin(dist_point_segment(a0, b0, b1), dist_point_segment(a1, b0, b1)));
}

typedef struct { int n; v2 p[ORC_MAX_V]; } poly_t;

/* geometry.cpp:56-64 */
static int point_in_convex(v2 p, const poly_t* poly) {
  for (int i = 0; i < poly->n; ++i) {
    const v2 a = poly->p[i], b = poly->p[(i + 1) % poly->n];
    if (cross(sub(b, a), sub(p, a)) < 0.0) return 0;
  }
  return 1;
}

/* geometry.cpp:66-79 */
static v2 polygon_centroid(const poly_t* poly) {
  double area2 = 0.0;
  v2 c = V(0.0, 0.0);
  for (int i = 0; i < poly->n; ++i) {
    const v2 a = poly->p[i], b = poly->p[(i + 1) % poly->n];
    const double w = cross(a, b);
    area2 += w;
    const v2 t = mul(add(a, b), w);
    c.x += t.x;
    c.y += t.y;
  }
  if (area2 == 0.0) return poly->n == 0 ? V(0.0, 0.0) : poly->p[0];
  return mul(c, 1.0 / (3.0 * area2));
}

/* geometry.cpp:81-85 */
static double support_extent(const poly_t* poly, v2 dir) {
  double best = -INFINITY;
  for (int i = 0; i < poly->n; ++i) best = dmax(best, dot(poly->p[i], dir));
  return best;
}

/* geometry.cpp:87-100 */
static v2 closest_point_on_polygon(v2 p, const poly_t* poly) {
  v2 best = V(0.0, 0.0);
  double best_d = INFINITY;
  for (int i = 0; i < poly->n; ++i) {
    const v2 q = closest_point_on_segment(p, poly->p[i], poly->p[(i + 1) % poly->n]);
    const double d = norm2(sub(p, q));
    if (d < best_d) {
      best_d = d;
      best = q;
    }
  }
  return best;
}

/* geometry.cpp:102-105 */
static double signed_dist_point_polygon(v2 p, const poly_t* poly) {
  const double d = norm(sub(p, closest_point_on_polygon(p, poly)));
  return point_in_convex(p, poly) ? -d : d;
}

typedef struct { double depth; v2 dir; v2 contact; } overlap_t;

/* geometry.cpp:107-115 */
static overlap_t disc_disc_overlap(v2 ca, double ra, v2 cb, double rb) {
  overlap_t o;
  const v2 d = sub(cb, ca);
  const double dist = norm(d);
  o.depth = ra + rb - dist;
  o.dir = dist > 0.0 ? mul(d, 1.0 / dist) : V(1.0, 0.0);
  o.contact = add(ca, mul(o.dir, ra));
  return o;
}

/* geometry.cpp:117-132 */
static overlap_t disc_polygon_overlap(v2 c, double r, const poly_t* poly) {
  overlap_t o;
  const v2 q = closest_point_on_polygon(c, poly);
  const v2 d = sub(q, c);
  const double dist = norm(d);
  o.contact = q;
  if (point_in_convex(c, poly)) {
    o.depth = r + dist;
  } else {
    o.depth = r - dist;
  }
  o.dir = dist > 0.0 ? mul(d, 1.0 / dist) : V(1.0, 0.0);
  return o;
}

/* geometry.cpp:137-152 */
static int sat_min_overlap(const poly_t* a, const poly_t* b, double* depth, v2* axis) {
  for (int i = 0; i < a->n; ++i) {
    const v2 edge = sub(a->p[(i + 1) % a->n], a->p[i]);
    const v2 normal = normalized(V(edge.y, -edge.x));
    const double a_max = support_extent(a, normal);
    const double b_min = -support_extent(b, neg(normal));
    const double o = a_max - b_min;
    if (o < *depth) {
      *depth = o;
      *axis = normal;
    }
    if (o <= 0.0) return 0;
  }
  return 1;
}

/* geometry.cpp:191-195 */
static int polygons_intersect(const poly_t* a, const poly_t* b) {
  double depth = INFINITY;
  v2 axis = V(0.0, 0.0);
  return sat_min_overlap(a, b, &depth, &axis) && sat_min_overlap(b, a, &depth, &axis);
}

/* geometry.cpp:176-184 */
static double dist_polygon_polygon(const poly_t* a, const poly_t* b) {
  if (polygons_intersect(a, b)) return 0.0;
  double best = INFINITY;
  for (int i = 0; i < a->n; ++i)
    for (int j = 0; j < b->n; ++j)
      best = dmin(best, dist_segment_segment(a->p[i], a->p[(i + 1) % a->n], b->p[j], b->p[(j + 1) % b->n]));
  return best;
}

/* geometry.cpp:156-174 */
static overlap_t polygon_polygon_overlap(const poly_t* a, const poly_t* b) {
  overlap_t o;
  o.contact = V(0.0, 0.0);
  double depth = INFINITY;
  v2 axis = V(0.0, 0.0);
  const int ab = sat_min_overlap(a, b, &depth, &axis);
  const int ba = ab && sat_min_overlap(b, a, &depth, &axis);
  if (!ab || !ba) {
    o.depth = -dist_polygon_polygon(a, b);
    o.dir = normalized(sub(polygon_centroid(b), polygon_centroid(a)));
    return o;
  }
  o.depth = depth;
  const v2 sep = sub(polygon_centroid(b), polygon_centroid(a));
  o.dir = dot(sep, axis) >= 0.0 ? axis : neg(axis);
  o.contact = mul(add(closest_point_on_polygon(polygon_centroid(b), a),
                      closest_point_on_polygon(polygon_centroid(a), b)), 0.5);
  return o;
}

/* ---------------- world (world.cpp) ---------------- */

/* world.cpp:32-37 */
static double bounding_radius(const orc_state* s, int i) {
  if (s->kind[i] == 0) return s->radius[i];
  double best = 0.0;
  for (int k = 0; k < s->nv[i]; ++k) best = dmax(best, norm(V(s->verts[i][k][0], s->verts[i][k][1])));
  return best;
}

/* world.cpp:57-62 */
static void world_polygon(const orc_state* s, int i, poly_t* out) {
  out->n = s->nv[i];
  const v2 pos = V(s->x[i], s->y[i]);
  for (int k = 0; k < s->nv[i]; ++k)
    out->p[k] = add(pos, rotated(V(s->verts[i][k][0], s->verts[i][k][1]), s->th[i]));
}

/* world.cpp:101-107 */
static double object_point_distance(const orc_state* s, int i, v2 p) {
  if (s->kind[i] == 0) return dmax(0.0, norm(sub(p, V(s->x[i], s->y[i]))) - s->radius[i]);
  poly_t poly;
  world_polygon(s, i, &poly);
  return dmax(0.0, signed_dist_point_polygon(p, &poly));
}

/* world.cpp:123-135 and push_sim.cpp:20-32 (identical) */
static overlap_t object_pair_overlap(const orc_state* s, int a, int b) {
  const int da = s->kind[a] == 0, db = s->kind[b] == 0;
  if (da && db) return disc_disc_overlap(V(s->x[a], s->y[a]), s->radius[a], V(s->x[b], s->y[b]), s->radius[b]);
  poly_t pa, pb;
  if (da) {
    world_polygon(s, b, &pb);
    return disc_polygon_overlap(V(s->x[a], s->y[a]), s->radius[a], &pb);
  }
  if (db) {
    world_polygon(s, a, &pa);
    overlap_t o = disc_polygon_overlap(V(s->x[b], s->y[b]), s->radius[b], &pa);
    o.dir = neg(o.dir);
    return o;
  }
  world_polygon(s, a, &pa);
  world_polygon(s, b, &pb);
  return polygon_polygon_overlap(&pa, &pb);
}

/* world.cpp:139-152 */
static double max_pairwise_penetration(const orc_state* s, int64_t* pfinal) {
  double worst = 0.0;
  for (int i = 0; i + 1 < s->n; ++i)
    for (int j = i + 1; j < s->n; ++j) {
      const double reach = bounding_radius(s, i) + bounding_radius(s, j);
      if (norm2(sub(V(s->x[i], s->y[i]), V(s->x[j], s->y[j]))) > reach * reach) continue;
      if (pfinal) ++*pfinal;
      worst = dmax(worst, object_pair_overlap(s, i, j).depth);
    }
  return worst;
}

/* world.cpp:154-164 */
static int collides_gripper_start(const orc_state* s, const double* push, const orc_params* p) {
  const double r = p->tip_r + p->tip_clear;
  const v2 q = V(push[0], push[1]);
  const double h = s->side / 2.0;
  if (q.x - r < -h || q.x + r > h || q.y - r < -h || q.y + r > h) return 1;
  for (int i = 0; i < s->n; ++i)
    if (object_point_distance(s, i, q) < r) return 1;
  return 0;
}

/* world.cpp:86-90 with Workspace::contains_point world.hpp:23-26 */
static int push_action_valid(const double* push, double dist, double side) {
  const double len = norm(sub(V(push[2], push[3]), V(push[0], push[1])));
  if (fabs(len - dist) > 1e-9) return 0;
  const double h = side / 2.0;
  const int s_in = push[0] > -h && push[0] < h && push[1] > -h && push[1] < h;
  const int e_in = push[2] > -h && push[2] < h && push[3] > -h && push[3] < h;
  return s_in && e_in;
}

/* world.cpp:166-191 */
static uint64_t state_digest(const orc_state* s) {
  uint64_t h = 1469598103934665603ull;
#define MIX(ptr, len)                                        \
  do {                                                       \
    const unsigned char* q_ = (const unsigned char*)(ptr);   \
    for (size_t k_ = 0; k_ < (len); ++k_) {                  \
      h ^= q_[k_];                                           \
      h *= 1099511628211ull;                                 \
    }                                                        \
  } while (0)
  const int32_t tgt = s->target;
  MIX(&tgt, 4);
  MIX(&s->side, 8);
  for (int i = 0; i < s->n; ++i) {
    const int32_t kind = s->kind[i];
    MIX(&kind, 4);
    MIX(&s->radius[i], 8);
    if (s->kind[i] != 0)
      for (int k = 0; k < s->nv[i]; ++k) {
        MIX(&s->verts[i][k][0], 8);
        MIX(&s->verts[i][k][1], 8);
      }
    MIX(&s->x[i], 8);
    MIX(&s->y[i], 8);
    MIX(&s->th[i], 8);
  }
#undef MIX
  return h;
}

/* ---------------- push simulator (push_sim.cpp) ---------------- */

/* push_sim.cpp:36-46 */
static void apply_contact_motion(orc_state* s, int i, v2 t, v2 contact, double gain) {
  s->x[i] += t.x;
  s->y[i] += t.y;
  if (s->kind[i] != 1 || gain == 0.0) return;
  const v2 lever = sub(contact, V(s->x[i], s->y[i]));
  const double lever2 = norm2(lever);
  if (lever2 < 1e-12) return;
  double dtheta = gain * cross(lever, t) / lever2;
  dtheta = dclamp(dtheta, -0.2, 0.2);
  s->th[i] = wrap_angle(s->th[i] + dtheta);
}

/* push_sim.cpp:13-18 */
static overlap_t tip_object_overlap(v2 tc, double tr, const orc_state* s, int i) {
  if (s->kind[i] == 0) return disc_disc_overlap(tc, tr, V(s->x[i], s->y[i]), s->radius[i]);
  poly_t poly;
  world_polygon(s, i, &poly);
  return disc_polygon_overlap(tc, tr, &poly);
}

/* push_sim.cpp:58-130.  Returns 0 ok, 1 start collision, 2 not converged;
 * *residual = final max pairwise penetration. */
static int resolve_push(orc_state* s, const double* push, const orc_params* p, double* residual,
                        orc_counts* cnt) {
  if (collides_gripper_start(s, push, p)) return 1;
  const int n = s->n;
  const v2 start = V(push[0], push[1]);
  const v2 end = V(push[2], push[3]);
  const v2 delta = mul(sub(end, start), 1.0 / p->substeps);
  const double sweep_reach = p->push_distance + p->tip_r;
  double br[ORC_MAX_OBJ];
  for (int i = 0; i < n; ++i) br[i] = bounding_radius(s, i);
  char active[ORC_MAX_OBJ];
  {
    double max_diam = 0.0;
    for (int i = 0; i < n; ++i) max_diam = dmax(max_diam, 2.0 * br[i]);
    const double reach = sweep_reach + 2.0 * max_diam;
    for (int i = 0; i < n; ++i) {
      const double d = dist_point_segment(V(s->x[i], s->y[i]), start, end);
      active[i] = d <= reach + br[i] ? 1 : 0;
    }
  }
  for (int step = 1; step <= p->substeps; ++step) {
    const v2 tc = add(start, mul(delta, (double)step));
    if (cnt) cnt->s++;
    for (int iter = 0; iter < p->max_iters; ++iter) {
      double max_pen = 0.0;
      for (int i = 0; i < n; ++i) {
        if (!active[i]) continue;
        const double reach = p->tip_r + br[i];
        if (cnt) cnt->tb++;
        if (norm2(sub(V(s->x[i], s->y[i]), tc)) > reach * reach) continue;
        if (cnt) cnt->tn++;
        const overlap_t o = tip_object_overlap(tc, p->tip_r, s, i);
        if (o.depth > 0.0) {
          if (cnt) cnt->ht++;
          apply_contact_motion(s, i, mul(o.dir, o.depth), o.contact, p->rotation_gain);
          max_pen = dmax(max_pen, o.depth);
        }
      }
      for (int i = 0; i + 1 < n; ++i) {
        if (!active[i]) continue;
        for (int j = i + 1; j < n; ++j) {
          if (!active[j]) continue;
          const double reach = br[i] + br[j];
          if (cnt) cnt->pb++;
          if (norm2(sub(V(s->x[i], s->y[i]), V(s->x[j], s->y[j]))) > reach * reach) continue;
          if (cnt) cnt->pn++;
          const overlap_t o = object_pair_overlap(s, i, j);
          if (o.depth > 0.0) {
            if (cnt) cnt->hp++;
            apply_contact_motion(s, i, mul(neg(o.dir), 0.5 * o.depth), o.contact, p->rotation_gain);
            apply_contact_motion(s, j, mul(o.dir, 0.5 * o.depth), o.contact, p->rotation_gain);
            max_pen = dmax(max_pen, o.depth);
          }
        }
      }
      /* clamp_to_boundary push_sim.cpp:48-54 */
      const double h = s->side / 2.0 - s->margin - 1e-9;
      for (int i = 0; i < n; ++i) {
        s->x[i] = dclamp(s->x[i], -h, h);
        s->y[i] = dclamp(s->y[i], -h, h);
      }
      if (max_pen <= p->eps_pen) break;
    }
  }
  const double final_pen = max_pairwise_penetration(s, cnt ? &cnt->pfinal : NULL);
  if (residual) *residual = final_pen;
  return final_pen > p->eps_pen ? 2 : 0;
}

/* ---------------- actions (actions.cpp) ---------------- */

/* actions.cpp:12-30 */
static double contour_radius(const orc_state* s, int i, v2 d) {
  if (s->kind[i] == 0) return s->radius[i];
  const v2 dl = rotated(d, -s->th[i]);
  double best = 0.0;
  const int n = s->nv[i];
  for (int k = 0; k < n; ++k) {
    const v2 a = V(s->verts[i][k][0], s->verts[i][k][1]);
    const v2 b = V(s->verts[i][(k + 1) % n][0], s->verts[i][(k + 1) % n][1]);
    const v2 e = sub(b, a);
    const double denom = cross(dl, e);
    if (fabs(denom) < 1e-15) continue;
    const double t = cross(a, e) / denom;
    const double sp = cross(a, dl) / denom;
    if (t > 0.0 && sp >= -1e-12 && sp <= 1.0 + 1e-12) best = dmax(best, t);
  }
  return best;
}

/* actions.cpp:51-73.  out capacity n * N_a * 4 doubles; returns count. */
static int sample_pushes(const orc_state* s, const orc_params* p, double* out) {
  const int na = p->pushes_per_object;
  if (na < 1) return 0;
  const double offset = p->tip_r + p->tip_clear + 1e-9;
  int count = 0;
  for (int i = 0; i < s->n; ++i) {
    const v2 center = V(s->x[i], s->y[i]);
    for (int k = 0; k < na; ++k) {
      const double angle = 2.0 * M_PI * k / na;
      const v2 d = V(cos(angle), sin(angle));
      const double cr = contour_radius(s, i, d);
      if (cr <= 0.0) continue;
      const v2 start = add(center, mul(d, cr + offset));
      const v2 dir = normalized(sub(center, start));
      const v2 end = add(start, mul(dir, p->push_distance));
      double push[4] = {start.x, start.y, end.x, end.y};
      if (!push_action_valid(push, p->push_distance, s->side)) continue;
      if (collides_gripper_start(s, push, p)) continue;
      memcpy(out + count * 4, push, sizeof push);
      ++count;
    }
  }
  return count;
}

typedef struct { poly_t a, b; v2 center; double extent; } fingers_t;

/* actions.cpp:75-111 */
static void grasp_fingers(const orc_state* s, const orc_params* p, int k, fingers_t* fp) {
  const int t = s->target;
  const double angle = 2.0 * M_PI * k / 16;
  const v2 u = V(cos(angle), sin(angle));
  const v2 v = perp(u);
  double lo_u, hi_u, lo_v, hi_v;
  if (s->kind[t] == 0) {
    const double cu = dot(V(s->x[t], s->y[t]), u);
    const double cv = dot(V(s->x[t], s->y[t]), v);
    lo_u = cu - s->radius[t];
    hi_u = cu + s->radius[t];
    lo_v = cv - s->radius[t];
    hi_v = cv + s->radius[t];
  } else {
    poly_t poly;
    world_polygon(s, t, &poly);
    hi_u = support_extent(&poly, u);
    lo_u = -support_extent(&poly, neg(u));
    hi_v = support_extent(&poly, v);
    lo_v = -support_extent(&poly, neg(v));
  }
  fp->extent = hi_u - lo_u;
  fp->center = add(mul(u, (lo_u + hi_u) / 2.0), mul(v, (lo_v + hi_v) / 2.0));
  const double ht = p->finger_thickness / 2.0;
  const double hw = p->finger_width / 2.0;
  for (int side = 0; side < 2; ++side) {
    const double off = side == 0 ? -(p->opening / 2.0 + ht) : p->opening / 2.0 + ht;
    const v2 c = add(fp->center, mul(u, off));
    poly_t* r = side == 0 ? &fp->a : &fp->b;
    r->n = 4;
    r->p[0] = sub(sub(c, mul(u, ht)), mul(v, hw));
    r->p[1] = sub(add(c, mul(u, ht)), mul(v, hw));
    r->p[2] = add(add(c, mul(u, ht)), mul(v, hw));
    r->p[3] = add(sub(c, mul(u, ht)), mul(v, hw));
  }
}

/* actions.cpp:32-39 */
static double rect_min_wall_clearance(const poly_t* rect, double side) {
  const double h = side / 2.0;
  double best = INFINITY;
  for (int i = 0; i < rect->n; ++i)
    best = dmin(best, dmin(h - fabs(rect->p[i].x), h - fabs(rect->p[i].y)));
  return best;
}

/* actions.cpp:41-47 */
static double rect_object_distance(const poly_t* rect, const orc_state* s, int i) {
  if (s->kind[i] == 0) {
    const double sd = signed_dist_point_polygon(V(s->x[i], s->y[i]), rect);
    return dmax(0.0, sd - s->radius[i]);
  }
  poly_t poly;
  world_polygon(s, i, &poly);
  return dist_polygon_polygon(rect, &poly);
}

/* actions.cpp:113-147.  Returns graspable flag. */
static int graspable(const orc_state* s, const orc_params* p, double* margin_out, double* bx,
                     double* by, int* bk) {
  double best_margin = -1.0;
  int best_k = -1;
  double best_x = 0.0, best_y = 0.0;
  for (int k = 0; k < 16; ++k) {
    fingers_t fp;
    grasp_fingers(s, p, k, &fp);
    if (!(fp.extent < p->opening - 2.0 * p->approach_clearance)) continue;
    if (dmin(rect_min_wall_clearance(&fp.a, s->side), rect_min_wall_clearance(&fp.b, s->side)) <= 0.0)
      continue;
    double margin = s->side;
    int feasible = 1;
    for (int i = 0; i < s->n; ++i) {
      if (i == s->target) continue;
      const double d = dmin(rect_object_distance(&fp.a, s, i), rect_object_distance(&fp.b, s, i));
      if (d <= 0.0) {
        feasible = 0;
        break;
      }
      margin = dmin(margin, d);
    }
    if (feasible && margin > best_margin) {
      best_margin = margin;
      best_k = k;
      best_x = fp.center.x;
      best_y = fp.center.y;
    }
  }
  if (margin_out) *margin_out = best_k >= 0 ? best_margin : 0.0;
  if (bx) *bx = best_x;
  if (by) *by = best_y;
  if (bk) *bk = best_k;
  return best_k >= 0 && best_margin >= p->margin_threshold;
}

/* ---------------- keyed RNG (rng.hpp) + libstdc++ mt19937_64 ---------------- */

static uint64_t splitmix64(uint64_t x) { /* rng.hpp:8-13 */
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
static uint64_t mix_keys(uint64_t seed, uint64_t a, uint64_t b) { /* rng.hpp:15-17 */
  return splitmix64(splitmix64(splitmix64(seed) ^ a) ^ b);
}

typedef struct { uint64_t mt[312]; int idx; } mt64;

static void mt_seed(mt64* g, uint64_t seed) { /* libstdc++ random.tcc mersenne_twister_engine::seed */
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ull * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}
static uint64_t mt_next(mt64* g) { /* random.tcc _M_gen_rand + operator() */
  const uint64_t UM = 0xffffffff80000000ull, LM = 0x7fffffffull, A = 0xb5026f5aa96619e9ull;
  if (g->idx >= 312) {
    int k;
    for (k = 0; k < 156; ++k) {
      const uint64_t y = (g->mt[k] & UM) | (g->mt[k + 1] & LM);
      g->mt[k] = g->mt[k + 156] ^ (y >> 1) ^ ((y & 1) ? A : 0);
    }
    for (; k < 311; ++k) {
      const uint64_t y = (g->mt[k] & UM) | (g->mt[k + 1] & LM);
      g->mt[k] = g->mt[k - 156] ^ (y >> 1) ^ ((y & 1) ? A : 0);
    }
    const uint64_t y = (g->mt[311] & UM) | (g->mt[0] & LM);
    g->mt[311] = g->mt[155] ^ (y >> 1) ^ ((y & 1) ? A : 0);
    g->idx = 0;
  }
  uint64_t z = g->mt[g->idx++];
  z ^= (z >> 29) & 0x5555555555555555ull;
  z ^= (z << 17) & 0x71d67fffeda60000ull;
  z ^= (z << 37) & 0xfff7eee000000000ull;
  z ^= (z >> 43);
  return z;
}
/* uniform_int_distribution<size_t>(0, n-1) via Lemire _S_nd
 * (/usr/include/c++/13/bits/uniform_int_dist.h:255-280, 313-321) */
static uint64_t mt_pick(mt64* g, uint64_t n) {
  unsigned __int128 prod = (unsigned __int128)mt_next(g) * n;
  uint64_t low = (uint64_t)prod;
  if (low < n) {
    const uint64_t thr = (0 - n) % n;
    while (low < thr) {
      prod = (unsigned __int128)mt_next(g) * n;
      low = (uint64_t)prod;
    }
  }
  return (uint64_t)(prod >> 64);
}

/* ---------------- flat-array loaders ---------------- */

static void load_state(orc_state* s, int e, int n, int n_tables, const int* kind, const double* radius,
                       const int* nv, const double* verts, const int* target, double side, double margin,
                       const double* poses) {
  const int t = n_tables == 1 ? 0 : e;
  s->n = n;
  s->target = target[t];
  s->side = side;
  s->margin = margin;
  for (int i = 0; i < n; ++i) {
    const int q = t * n + i;
    s->kind[i] = kind[q];
    s->radius[i] = radius[q];
    s->nv[i] = nv ? nv[q] : 0;
    for (int k = 0; k < ORC_MAX_V; ++k) {
      s->verts[i][k][0] = verts ? verts[(q * ORC_MAX_V + k) * 2] : 0.0;
      s->verts[i][k][1] = verts ? verts[(q * ORC_MAX_V + k) * 2 + 1] : 0.0;
    }
    s->x[i] = poses[(e * n + i) * 3];
    s->y[i] = poses[(e * n + i) * 3 + 1];
    s->th[i] = poses[(e * n + i) * 3 + 2];
  }
}

static void store_poses(const orc_state* s, double* out) {
  for (int i = 0; i < s->n; ++i) {
    out[i * 3] = s->x[i];
    out[i * 3 + 1] = s->y[i];
    out[i * 3 + 2] = s->th[i];
  }
}

#define SHAPE_ARGS int n, int n_tables, const int *kind, const double *radius, const int *nv, \
                   const double *verts, const int *target, double side, double margin
#define SHAPE_PASS n, n_tables, kind, radius, nv, verts, target, side, margin

/* ---------------- exported entry points ---------------- */

/* batch_resolve (push_sim.cpp:132-152), element-wise.  counts: [E][8] or NULL. */
int orc_batch_resolve(int E, SHAPE_ARGS, const double* poses, const double* pushes, const orc_params* p,
                      double* poses_out, int* status, double* residual, int64_t* counts) {
  for (int e = 0; e < E; ++e) {
    orc_state s;
    load_state(&s, e, SHAPE_PASS, poses);
    orc_counts c;
    memset(&c, 0, sizeof c);
    double res = 0.0;
    const int st = resolve_push(&s, pushes + e * 4, p, &res, counts ? &c : NULL);
    status[e] = st;
    if (residual) residual[e] = st == 1 ? 0.0 : res;
    if (st == 0) store_poses(&s, poses_out + (size_t)e * n * 3);
    else memset(poses_out + (size_t)e * n * 3, 0, sizeof(double) * n * 3);
    if (counts) {
      int64_t* q = counts + (size_t)e * 8;
      q[0] = c.tb; q[1] = c.tn; q[2] = c.ht; q[3] = c.pb; q[4] = c.pn; q[5] = c.hp; q[6] = c.s; q[7] = c.pfinal;
    }
  }
  return 0;
}

int orc_state_digest(int E, SHAPE_ARGS, const double* poses, uint64_t* out) {
  for (int e = 0; e < E; ++e) {
    orc_state s;
    load_state(&s, e, SHAPE_PASS, poses);
    out[e] = state_digest(&s);
  }
  return 0;
}

int orc_sample_pushes(int e, SHAPE_ARGS, const double* poses, const orc_params* p, double* out) {
  orc_state s;
  load_state(&s, e, SHAPE_PASS, poses);
  return sample_pushes(&s, p, out);
}

int orc_graspable(int e, SHAPE_ARGS, const double* poses, const orc_params* p, double* margin_out,
                  double* bx, double* by, int* bk) {
  orc_state s;
  load_state(&s, e, SHAPE_PASS, poses);
  return graspable(&s, p, margin_out, bx, by, bk);
}

int orc_keyed_picks(uint64_t seed, uint64_t iter, uint64_t env, int count, uint64_t n, uint64_t* out) {
  mt64 g;
  mt_seed(&g, mix_keys(seed, iter, env));
  for (int k = 0; k < count; ++k) out[k] = mt_pick(&g, n);
  return 0;
}

uint64_t orc_mix_keys(uint64_t seed, uint64_t a, uint64_t b) { return mix_keys(seed, a, b); }

/* ---------------- rollouts + lockstep (mcts.cpp:121-171, pmbs.cpp:133-234) ---------------- */

typedef struct {
  orc_state s;
  int pushes, cap, done, by_grasp;
  double reward;
} cursor_t;

/* RolloutCursor ctor mcts.cpp:121-140 */
static void cursor_init(cursor_t* c, const orc_state* base, const double* node_poses, const int* meta,
                        int depth_cap, const orc_params* p) {
  c->s = *base;
  for (int i = 0; i < base->n; ++i) {
    c->s.x[i] = node_poses[i * 3];
    c->s.y[i] = node_poses[i * 3 + 1];
    c->s.th[i] = node_poses[i * 3 + 2];
  }
  c->pushes = meta[0];
  c->cap = depth_cap;
  c->done = 0;
  c->by_grasp = 0;
  c->reward = 0.0;
  if (meta[1]) {
    c->done = 1;
    c->by_grasp = 1;
    c->reward = pow(p->gamma, (double)meta[0]);
  } else if (meta[2]) {
    c->done = 1;
  } else if (c->pushes >= c->cap) {
    c->done = 1;
  }
}

/* RolloutCursor::step mcts.cpp:142-171 */
static void cursor_step(cursor_t* c, mt64* g, const orc_params* p, double* scratch, int64_t* ctr) {
  if (c->done) return;
  const int na = sample_pushes(&c->s, p, scratch);
  if (na == 0) {
    c->done = 1;
    c->reward = 0.0;
    return;
  }
  const uint64_t k = mt_pick(g, (uint64_t)na);
  double res;
  if (ctr) ctr[3]++;
  if (resolve_push(&c->s, scratch + k * 4, p, &res, NULL) != 0) {
    c->done = 1;
    c->reward = 0.0;
    return;
  }
  ++c->pushes;
  if (graspable(&c->s, p, NULL, NULL, NULL, NULL)) {
    c->done = 1;
    c->by_grasp = 1;
    c->reward = pow(p->gamma, (double)c->pushes);
    return;
  }
  if (c->pushes >= c->cap) {
    c->done = 1;
    c->reward = 0.0;
  }
}

/* batch_simulate -> lockstep_simulate (pmbs.cpp:207-234, 133-205) over
 * n_nodes node states sharing one shape table.  node_meta[i] = {depth,
 * graspable, dead}.  counters (4): rollout steps, rounds, re-purposes,
 * resolve calls. */
int orc_simulate(SHAPE_ARGS, const double* node_poses, const int* node_meta, int n_nodes, int n_envs,
                 int leaf_parallel, uint64_t seed, uint64_t iteration, int depth_cap, const orc_params* p,
                 double* rewards, int64_t* counters) {
  if (n_nodes <= 0) return 0;
  if (n_envs < n_nodes) return -1;
  orc_state base;
  load_state(&base, 0, SHAPE_PASS, node_poses);
  const int used = leaf_parallel ? n_envs : n_nodes;
  int* env_node = (int*)malloc(sizeof(int) * used);
  char* harvested = (char*)calloc(used, 1);
  cursor_t* cur = (cursor_t*)malloc(sizeof(cursor_t) * used);
  mt64* gens = (mt64*)malloc(sizeof(mt64) * n_envs);
  double* scratch = (double*)malloc(sizeof(double) * 4 * n * p->pushes_per_object + 4);
  int64_t ctr[4] = {0, 0, 0, 0};
  for (int e = 0; e < n_envs; ++e) mt_seed(&gens[e], mix_keys(seed, iteration, (uint64_t)e));
  {
    const int b = used / n_nodes, rem = used % n_nodes;
    int e = 0;
    for (int i = 0; i < n_nodes; ++i) {
      const int cnt = b + (i < rem ? 1 : 0);
      for (int k = 0; k < cnt; ++k) env_node[e++] = i;
    }
  }
  for (int e = 0; e < used; ++e)
    cursor_init(&cur[e], &base, node_poses + (size_t)env_node[e] * n * 3, node_meta + env_node[e] * 3,
                depth_cap, p);
  for (int i = 0; i < n_nodes; ++i) rewards[i] = 0.0;
  int round = 0;
  for (;;) {
    /* harvest_and_repurpose pmbs.cpp:165-187 */
    for (int e = 0; e < used; ++e) {
      if (harvested[e] || !cur[e].done) continue;
      harvested[e] = 1;
      const int nd = env_node[e];
      rewards[nd] = dmax(rewards[nd], cur[e].reward);
      if (!leaf_parallel || !cur[e].by_grasp) continue;
      int best_node = -1, best_work = 0;
      for (int i = 0; i < n_nodes; ++i) {
        int w = 0; /* remaining_work pmbs.cpp:157-163 */
        for (int f = 0; f < used; ++f)
          if (env_node[f] == i && !cur[f].done) w += cur[f].cap - cur[f].pushes;
        if (w > best_work) {
          best_work = w;
          best_node = i;
        }
      }
      if (best_node >= 0) {
        env_node[e] = best_node;
        cursor_init(&cur[e], &base, node_poses + (size_t)best_node * n * 3, node_meta + best_node * 3,
                    depth_cap, p);
        harvested[e] = 0;
        ctr[2]++;
      }
    }
    int any = 0;
    for (int e = 0; e < used; ++e) {
      if (cur[e].done) continue;
      any = 1;
      cursor_step(&cur[e], &gens[e], p, scratch, ctr);
      ctr[0]++;
    }
    if (!any) break;
    ++round;
  }
  ctr[1] = round;
  if (counters) memcpy(counters, ctr, sizeof ctr);
  free(env_node);
  free(harvested);
  free(cur);
  free(gens);
  free(scratch);
  return 0;
}
