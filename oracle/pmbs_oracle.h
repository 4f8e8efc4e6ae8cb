/*
 * pmbs_oracle.h — TEST INFRASTRUCTURE ONLY: a plain-C CPU restatement of the
 * reference's batched-rollout hot path (arxiv 2207.06649 "pushplan",
 * /root/reference/proj/core).  Used only by tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg as the CHECKER; the product never links it.
 * Pinned bit-for-bit against the compiled reference (oracle/_ref) by
 * tests/test_oracle.py and against the committed golden fixtures in
 * tests/golden/.
 */
#ifndef PMBS_ORACLE_H_
#define PMBS_ORACLE_H_

#include <stdint.h>

#define ORC_MAX_OBJ 32
#define ORC_MAX_V 8

typedef struct orc_state {
  int n;
  int target;
  double side;
  double margin;
  int kind[ORC_MAX_OBJ];
  double radius[ORC_MAX_OBJ];
  int nv[ORC_MAX_OBJ];
  double verts[ORC_MAX_OBJ][ORC_MAX_V][2];
  double x[ORC_MAX_OBJ], y[ORC_MAX_OBJ], th[ORC_MAX_OBJ];
} orc_state;

typedef struct orc_params {
  double tip_r, tip_clear;
  double push_distance;
  int substeps, max_iters;
  double eps_pen, rotation_gain;
  double finger_width, finger_thickness, opening, approach_clearance;
  double gamma;
  int pushes_per_object;
  double margin_threshold;
} orc_params;

/* counters for the algorithmic-work formula */
typedef struct orc_counts {
  int64_t tb, tn, ht, pb, pn, hp, s, pfinal;
} orc_counts;

#endif
