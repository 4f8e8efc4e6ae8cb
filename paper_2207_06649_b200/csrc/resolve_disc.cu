// resolve_disc.cu — the disc-scene physics kernel (kernel #1 fast path):
// resolve_push (push_sim.cpp:58-130) for batches whose objects are all discs
// (every proj/cases disc scene, the C2 / C4 workloads), bit-identical to the
// reference.
//
// Why a second kernel: the straight transcription (kernels.cu) spends ~90 %
// of its algorithmic FP64 work in broad-phase tests (7 ops each, uniform
// across lanes) but executes the rare narrow tests (sqrt + div, ~2 % of
// pairs) whenever ANY lane of the warp needs them, and pays address
// arithmetic on every shared-memory pose access.  Here, per projection
// iteration and per lane (= environment):
//
//   1. tip broad phase over all objects from FLOAT registers on the packed
//      FP32x2 pipe (FFMA2 / FADD2 / FMUL2, two objects per instruction; a
//      conservative superset of the FP64 test, see below) -> candidates;
//   2. tip narrow tests in a loop over the set bits (exact FP64 poses in
//      shared memory, dynamic index), each re-tested first with the
//      reference's FP64 broad expression — objects are independent in the
//      tip loop (push_sim.cpp:90-100), so any order is exact;
//   3. pair broad phase over all i<j, packed FP32x2 -> flat pair bitmask
//      (+ a `near` mask for the re-queue filter);
//   4. pair narrow tests in lexicographic order over the set bits, each
//      re-tested exactly in FP64 first.  A hit on (i,j) moves i and j, so
//      every LATER pair touching i or j is re-queued for evaluation (its
//      broad result is stale); a pair not re-queued has unchanged inputs, so
//      its broad result still holds.  This reproduces the reference's
//      in-place Gauss-Seidel sweep (push_sim.cpp:101-117) exactly while
//      running ~1 narrow test per lane per iteration;
//   5. clamp (push_sim.cpp:48-54): a conservative float test, the exact
//      clamp from shared memory for objects near a wall.
//
// Float filters: per environment, margin m = 2^-15 B (B bounds every
// coordinate, radius and push endpoint); float rounding moves a distance by
// < 2^-20 B, so a float test with radii padded by m/2 accepts everything the
// FP64 test accepts, and every float candidate is re-tested in FP64 — the
// candidate sequence, hence every result bit, is the reference's.
//
// The (substep, iteration) double loop is flattened per lane and lanes are
// persistent: a lane that finishes its environment fetches the next one, so
// warps stay full until the batch drains (no per-warp max-iteration tail).
// Streamed host batches (ctx.cu batch_resolve_streamed) add per-slice ready
// flags / done counters and, for pinned outputs, warp-coalesced writes of
// each finished env's record straight to host memory.
#include <cuda_runtime.h>

#include <climits>
#include <utility>

#include "kernels.cuh"

namespace ppg {

namespace {

constexpr int kDB = 128;  // threads per block

// Compile-time loops: the body receives std::integral_constant<int, I>, so
// every register-array index below is a constant expression and the arrays
// stay in registers.
template <class F, int... Is>
PPG_DI void static_for_impl(F&& f, std::integer_sequence<int, Is...>) {
  (f(std::integral_constant<int, Is>{}), ...);
}
template <int N, class F>
PPG_DI void static_for(F&& f) {
  static_for_impl(f, std::make_integer_sequence<int, N>{});
}

// lexicographic pair p of n objects -> (i, j), evaluated at compile time
__host__ __device__ constexpr int pair_i(int p, int n) {
  int i = 0;
  while (p >= n - 1 - i) {
    p -= n - 1 - i;
    ++i;
  }
  return i;
}
__host__ __device__ constexpr int pair_j(int p, int n) {
  int i = 0;
  while (p >= n - 1 - i) {
    p -= n - 1 - i;
    ++i;
  }
  return i + 1 + p;
}

template <int W>
struct Mask {
  uint64_t w[W];
  PPG_DI void clear() {
#pragma unroll
    for (int k = 0; k < W; ++k) w[k] = 0;
  }
  PPG_DI bool any() const {
    uint64_t o = 0;
#pragma unroll
    for (int k = 0; k < W; ++k) o |= w[k];
    return o != 0;
  }
  // pops the lowest set bit; returns its index (mask must be non-empty).
  // Branch-free over words (constant indices only) so the mask stays in
  // registers.
  PPG_DI int pop() {
    int idx = -1;
    bool done = false;
#pragma unroll
    for (int k = 0; k < W; ++k) {
      const bool take = !done && w[k] != 0;
      const int b = __ffsll(static_cast<long long>(w[k])) - 1;
      idx = take ? k * 64 + b : idx;
      w[k] = take ? (w[k] & (w[k] - 1)) : w[k];
      done = done || take;
    }
    return idx;
  }
  PPG_DI void assign(int q, bool v) {
#pragma unroll
    for (int k = 0; k < W; ++k) {
      const uint64_t bit = (q >> 6) == k ? (1ull << (q & 63)) : 0ull;
      w[k] = v ? (w[k] | bit) : (w[k] & ~bit);
    }
  }
  // this |= ((a | b) & m & bits strictly above p)
  PPG_DI void or_above(const uint64_t* a, const uint64_t* b, const Mask& m, int p) {
    const int pw = p >> 6, pb = p & 63;
#pragma unroll
    for (int k = 0; k < W; ++k) {
      const uint64_t above = k > pw ? ~0ull : (k < pw ? 0ull : (pb == 63 ? 0ull : (~0ull << (pb + 1))));
      w[k] |= (a[k] | b[k]) & m.w[k] & above;
    }
  }
};

constexpr double kNear = 0.002;  // metres, the re-queue filter margin
constexpr int kFixK = 6;         // check for a fixed point from this iteration of a substep on

// Streamed batches: is the slice holding env e resident?  (The copy stream
// writes `epoch` into its flag after the slice's copies.)
PPG_DI bool slice_ready(const ResolveArgs& a, int e) {
  const unsigned* f = a.ready + e / a.slice_envs;
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
  return v == a.epoch;
}

// Streamed batches: env e's outputs are written; count it for its slice.
PPG_DI void slice_done(const ResolveArgs& a, int e) {
  __threadfence();
  atomicAdd(a.done + e / a.slice_envs, 1u);
}

PPG_DI double fclampd(double v, double lo, double hi) {
  // == std::clamp(v, lo, hi) for non-NaN v (positions are finite)
  return fmin(fmax(v, lo), hi);
}

}  // namespace

template <int NMAX, bool kFix>
__global__ void __launch_bounds__(kDB, NMAX <= 10 ? 4 : NMAX <= 16 ? 3 : 2) resolve_disc_kernel(const __grid_constant__ SimConst C, ResolveArgs a,
                                                               int* next_env) {
  constexpr int P = NMAX * (NMAX - 1) / 2;
  constexpr int W = (P + 63) / 64;
  // dynamic shared memory (disc_smem): doubles [x | y | r | theta][NMAX][kDB]
  // (theta only for NMAX <= 14), then the float shadows [xf | yf][NMAX][kDB]
  // of x / y, written together with them (no conversions on the refreshes)
  extern __shared__ double dsm[];
  constexpr int kDPlanes = NMAX <= 14 ? 4 : 3;
  __shared__ uint16_t pij[P];  // i | j << 8
  __shared__ uint64_t omask[NMAX][W];  // pairs touching object k

  const int tid = threadIdx.x;
  for (int q = tid; q < NMAX * W; q += kDB) (&omask[0][0])[q] = 0;
  __syncthreads();
  if (tid == 0) {
    int p = 0;
    for (int i = 0; i < NMAX; ++i)
      for (int j = i + 1; j < NMAX; ++j, ++p) {
        pij[p] = static_cast<uint16_t>(i | (j << 8));
        omask[i][p >> 6] |= 1ull << (p & 63);
        omask[j][p >> 6] |= 1ull << (p & 63);
      }
  }
  __syncthreads();

  const int n = C.n;
  const double tr = C.tip_r;
  const double hcl = C.side / 2.0 - C.margin - 1e-9;
  double* const xl = dsm + tid;
  double* const yl = dsm + NMAX * kDB + tid;
  double* const rl = dsm + 2 * NMAX * kDB + tid;
  double* const tl = dsm + 3 * NMAX * kDB + tid;  // (kDPlanes == 4 only)
  float* const xs = reinterpret_cast<float*>(dsm + kDPlanes * NMAX * kDB) + tid;
  float* const ys = xs + NMAX * kDB;

  // Float copies of the positions and margin-padded radii (r + m/2) for the
  // broad-phase filters: every float test is a strict superset of the
  // reference's FP64 test (margin m, set per environment), and every
  // candidate is re-tested exactly in FP64 from shared memory, so results
  // are unchanged while the uniform all-pairs work runs on the FP32 pipe.
  // Stored as float2 pairs (objects 2m, 2m+1) so the broad phases run on the
  // packed FP32x2 pipe (sm_100 FFMA2/FADD2/FMUL2): XF(i) / YF(i) / RM(i).
  constexpr int NP = (NMAX + 1) / 2;
  float2 xp[NP], yp[NP], rp[NP];
#define XF(i) ((((i) & 1) ? xp[(i) >> 1].y : xp[(i) >> 1].x))
#define YF(i) ((((i) & 1) ? yp[(i) >> 1].y : yp[(i) >> 1].x))
#define RM(i) ((((i) & 1) ? rp[(i) >> 1].y : rp[(i) >> 1].x))
#pragma unroll
  for (int k = 0; k < NP; ++k) xp[k] = yp[k] = rp[k] = make_float2(0.f, 0.f);
  float trm = 0.f, hclf = 0.f;
  double fx0[NMAX], fy0[NMAX];  // fixed-point check copies (local memory)
  uint32_t active = 0;
  Mask<W> pact;  // pairs with both objects active
  V2 start{0.0, 0.0}, delta{0.0, 0.0};
  int step = 0, iter = 0;
  int budget_left = 0;  // wave rounds (kFix): iterations left in this launch
  const int E = a.E_dev ? *a.E_dev : a.E;
  // First environments: an even share per block (`per` <= kDB), so a full
  // wave of blocks (the launch fills every SM equally) gives every SM the
  // same number of environments; the rest are fetched with one atomic each.
  const int per = min(kDB, (E + static_cast<int>(gridDim.x) - 1) / static_cast<int>(gridDim.x));
  const int total_threads = gridDim.x * per;
  // Streamed batches: warp-major (warp w of every block before warp w+1; 32
  // consecutive envs per warp), so the first slices' envs are spread over
  // every SM and a warp's lanes mostly share one slice.
  int e = INT_MAX;
  if (tid < per) {
    if (a.ready) {
      const int w = tid >> 5, lanes = min(32, per - (w << 5));
      e = (w << 5) * static_cast<int>(gridDim.x) + static_cast<int>(blockIdx.x) * lanes + (tid & 31);
    } else {
      e = blockIdx.x * per + tid;
    }
  }
  const int rs_i = a.rad_env_major ? 1 : a.S.T;  // radius strides (object, table)
  const int rs_t = a.rad_env_major ? n : 1;
  int ee = e;
  bool have = false;
  bool need_init = true;
  bool pending = false;  // streamed: this lane's next env is in a slice not yet resident
  int zc_env = 0, zc_kind = 0, zc_st = 0;  // zc_out: finished env awaiting its flush (1 poses, 2 zeros)
  double zc_res = 0.0;
  const int lane = tid & 31;
  double* const xw = dsm + (tid - lane);  // this warp's shared-memory columns
  double* const yw = dsm + NMAX * kDB + (tid - lane);
  double* const tw = dsm + 3 * NMAX * kDB + (tid - lane);

  while (true) {
    // ---- zc_out: the warp writes each just-finished env's poses to host
    // memory, one contiguous [n][3] record per env (consecutive lanes ->
    // consecutive doubles), before the lane's columns are re-used
    if (a.zc_out) {
      unsigned m = __ballot_sync(0xffffffffu, zc_kind != 0);
      while (m) {
        const int src = __ffs(m) - 1;
        m &= m - 1;
        const int se = __shfl_sync(0xffffffffu, zc_env, src);
        const int sk = __shfl_sync(0xffffffffu, zc_kind, src);
        const int sst = __shfl_sync(0xffffffffu, zc_st, src);
        const double sres = __shfl_sync(0xffffffffu, zc_res, src);
        double* dst = a.poses_out + static_cast<size_t>(se) * n * 3;
        for (int q = lane; q < n * 3; q += 32) {
          const int obj = q / 3, c = q - 3 * obj;
          double v = 0.0;
          if (sk == 1)
            v = c < 2 || kDPlanes == 4 ? (c == 0 ? xw : c == 1 ? yw : tw)[obj * kDB + src]
                                       : __ldcg(a.poses_in + static_cast<size_t>(se) * n * 3 + q);
          dst[q] = v;
        }
        if (lane == 0) a.status[se] = sst;
        if (lane == 1 && a.residual) a.residual[se] = sres;
      }
      zc_kind = 0;
    }
    // ---- environment init: load, precondition, active mask (push_sim.cpp:58-82)
    if (need_init) {
      need_init = false;
      have = false;
      pending = false;
      while (e < E) {
        if (a.ready && !slice_ready(a, e)) {  // retried on the next pass; the warp runs on
          pending = true;
          need_init = true;
          break;
        }
        ee = a.idx ? a.idx[e] : e;  // environment slot (indirection for the lockstep engine)
        const double* src = a.poses_in + static_cast<size_t>(ee) * n * 3;
        const int t = a.S.T == 1 ? 0 : ee;
        // poses -> shared memory (the exact FP64 copy) and float registers
        // (broad-phase filters only); B bounds every coordinate / radius
        double B = C.side / 2.0 + C.tip_r;
        static_for<NMAX>([&](auto ic) {
          constexpr int i = decltype(ic)::value;
          const bool real = i < n;
          // inputs are read once, through L2 (.cg: streamed slices are
          // written by the copy engine while the kernel runs)
          const double xi = real ? __ldcg(src + i * 3) : 0.0;
          const double yi = real ? __ldcg(src + i * 3 + 1) : 0.0;
          const double ri = real ? __ldcg(a.S.rad + static_cast<size_t>(i) * rs_i + static_cast<size_t>(t) * rs_t) : 0.0;
          xl[i * kDB] = xi;
          yl[i * kDB] = yi;
          rl[i * kDB] = ri;
          XF(i) = static_cast<float>(xi);
          YF(i) = static_cast<float>(yi);
          xs[i * kDB] = XF(i);
          ys[i * kDB] = YF(i);
          if (kDPlanes == 4) tl[i * kDB] = real ? __ldcg(src + i * 3 + 2) : 0.0;
          B = fmax(B, fmax(fmax(fabs(xi), fabs(yi)), 4.0 * ri));
        });
        const double* pu = a.pushes + static_cast<size_t>(ee) * 4;
        start = V2{__ldcg(pu), __ldcg(pu + 1)};
        const V2 end{__ldcg(pu + 2), __ldcg(pu + 3)};
        B = fmax(B, fmax(fmax(fabs(start.x), fabs(start.y)), fmax(fabs(end.x), fabs(end.y))));
        // filter margin: float rounding of coordinates <= B moves a distance
        // by < 2^-20 B; 2^-15 B keeps the float tests strict supersets
        const double m = B * 0x1p-15;
        static_for<NMAX>([&](auto ic) {
          constexpr int i = decltype(ic)::value;
          RM(i) = static_cast<float>(rl[i * kDB] + 0.5 * m);
        });
        trm = static_cast<float>(tr + 0.5 * m);
        hclf = static_cast<float>(hcl - m);
        int rsi = -1;  // wave rounds: saved progress of a yielded push
        if constexpr (kFix) {
          if (a.resume_si) {
            rsi = __ldcg(a.resume_si + ee);
            budget_left = a.budget_dev ? __ldcg(a.budget_dev) : a.budget;
          }
        }
        if (kFix && rsi >= 0) {  // resume: progress saved at the yield, the precondition already passed
          delta = (end - start) * (1.0 / C.substeps);
          active = __ldcg(a.resume_active + ee);
          pact.clear();
          static_for<P>([&](auto pc) {
            constexpr int p = decltype(pc)::value;
            constexpr int i = pair_i(p, NMAX), j = pair_j(p, NMAX);
            if ((active >> i & 1u) && (active >> j & 1u)) pact.w[p >> 6] |= 1ull << (p & 63);
          });
          step = rsi >> 8;
          iter = rsi & 0xff;
          have = true;
          break;
        }
        // collides_gripper_start (world.cpp:154-164)
        bool collide = false;
        {
          const double rr = C.tip_r + C.tip_clear;
          const double h = C.side / 2.0;
          if (start.x - rr < -h || start.x + rr > h || start.y - rr < -h || start.y + rr > h) collide = true;
          for (int i = 0; i < n; ++i)
            if (dmax(0.0, norm(start - V2{xl[i * kDB], yl[i * kDB]}) - rl[i * kDB]) < rr) collide = true;
        }
        if (collide) {
          if (a.done) slice_done(a, e);
          if constexpr (kFix) {
            if (a.fin_list) a.fin_list[atomicAdd(a.fin_count, 1)] = ee;  // wave rounds: post pending
          }
          const int next = atomicAdd(next_env, 1) + total_threads;
          // zc_out: queued for the warp's coalesced flush only while this lane
          // has a next env (it then stays in the loop, so the flush at the loop
          // top runs); the batch's last envs of a lane, and a second queued
          // record, are written by the lane itself
          if (a.zc_out && zc_kind == 0 && next < E) {
            zc_env = ee;
            zc_kind = 2;
            zc_st = 1;
            zc_res = 0.0;
          } else {
            a.status[ee] = 1;
            if (a.residual) a.residual[ee] = 0.0;
            double* out = a.poses_out + static_cast<size_t>(ee) * n * 3;
            for (int i = 0; i < n * 3; ++i) out[i] = 0.0;
          }
          e = next;
          continue;
        }
        delta = (end - start) * (1.0 / C.substeps);
        double max_diam = 0.0;
        for (int i = 0; i < n; ++i) max_diam = dmax(max_diam, 2.0 * rl[i * kDB]);
        const double reach = (C.push_distance + C.tip_r) + 2.0 * max_diam;
        active = 0;
        for (int i = 0; i < n; ++i)
          if (dist_point_segment(V2{xl[i * kDB], yl[i * kDB]}, start, end) <= reach + rl[i * kDB]) active |= 1u << i;
        pact.clear();
        static_for<P>([&](auto pc) {
          constexpr int p = decltype(pc)::value;
          constexpr int i = pair_i(p, NMAX), j = pair_j(p, NMAX);
          if ((active >> i & 1u) && (active >> j & 1u)) pact.w[p >> 6] |= 1ull << (p & 63);
        });
        step = 1;
        iter = 0;
        if (C.max_iters < 1) step = C.substeps + 1;
        have = true;
        break;
      }
    }
    if (!__any_sync(0xffffffffu, have || pending)) break;
    if (!have) {
      // (the wait is bounded on the host: ctx.cu wait_streamed releases the
      // flags if the physics launch outlives PPG_STREAM_TIMEOUT_S; a kernel-side
      // poll counter measured 8.6 % slower on the C2 step)
      if (pending) __nanosleep(200);
      continue;
    }

    if (step > C.substeps) {
      // ---- final all-pairs penetration check + output (push_sim.cpp:123-128,
      // world.cpp:139-152).  Registers hold the final poses (kept in sync by
      // the clamp step).  max is order-free, so the candidates can be visited
      // in any order.
      Mask<W> fin;
      fin.clear();
      static_for<P>([&](auto pc) {
        constexpr int p = decltype(pc)::value;
        constexpr int i = pair_i(p, NMAX), j = pair_j(p, NMAX);
        const float dx = XF(i) - XF(j), dy = YF(i) - YF(j);
        const float rr = RM(i) + RM(j);
        if (j < n && !(__fmaf_rn(dx, dx, dy * dy) > rr * rr)) fin.w[p >> 6] |= 1ull << (p & 63);
      });
      double worst = 0.0;
      while (fin.any()) {
        const int ij = pij[fin.pop()];
        const int i = ij & 0xff, j = ij >> 8;
        const double bx = xl[i * kDB] - xl[j * kDB], by = yl[i * kDB] - yl[j * kDB];
        const double rr = rl[i * kDB] + rl[j * kDB];
        const double d2 = bx * bx + by * by;
        if (d2 > rr * rr) continue;  // the exact FP64 filter
        worst = dmax(worst, rr - sqrt(d2));  // == norm(pos_j - pos_i)
      }
      const int st = worst > C.eps_pen ? 2 : 0;
      double* out = a.poses_out + static_cast<size_t>(ee) * n * 3;
      if (a.zc_out && zc_kind == 0) {  // flushed by the warp at the top of the loop
        zc_env = ee;
        zc_kind = st == 0 ? 1 : 2;
        zc_st = st;
        zc_res = worst;
      } else {
        a.status[ee] = st;
        if (a.residual) a.residual[ee] = worst;
        if (st == 0) {
          for (int i = 0; i < n; ++i) {
            out[i * 3] = xl[i * kDB];
            out[i * 3 + 1] = yl[i * kDB];
            out[i * 3 + 2] = kDPlanes == 4 ? tl[i * kDB]  // discs never rotate (in place: same value)
                                            : __ldcg(a.poses_in + (static_cast<size_t>(ee) * n + i) * 3 + 2);
          }
        } else {
          for (int i = 0; i < n * 3; ++i) out[i] = 0.0;
        }
      }
      if (a.done) slice_done(a, e);
      if constexpr (kFix) {
        if (a.fin_list) a.fin_list[atomicAdd(a.fin_count, 1)] = ee;  // wave rounds: post pending
      }
      e = atomicAdd(next_env, 1) + total_threads;
      need_init = true;
      have = false;
      continue;
    }

    // ---- one projection iteration of substep `step` (push_sim.cpp:87-120)
    const V2 tc = start + delta * static_cast<double>(step);
    double max_pen = 0.0;
    // fixed-point check for long substeps (jams): the iteration-start state,
    // in local memory (runtime-indexed, so it never costs registers)
    if (kFix && C.fixpoint && iter >= kFixK) {
#pragma unroll 1
      for (int k = 0; k < n; ++k) {
        fx0[k] = xl[k * kDB];
        fy0[k] = yl[k * kDB];
      }
    }
    // 1-2. tip vs objects (push_sim.cpp:90-100)
    uint32_t tcand = 0;
    {
      const float tcx = static_cast<float>(tc.x), tcy = static_cast<float>(tc.y);
      const float2 tx2 = make_float2(tcx, tcx), ty2 = make_float2(tcy, tcy), tr2 = make_float2(trm, trm);
      const float2 m1 = make_float2(-1.f, -1.f);
      static_for<NP>([&](auto mc) {
        constexpr int mm = decltype(mc)::value;
        const float2 dx = __ffma2_rn(tx2, m1, xp[mm]), dy = __ffma2_rn(ty2, m1, yp[mm]);
        const float2 reach = __fadd2_rn(tr2, rp[mm]);
        const float2 d2 = __ffma2_rn(dx, dx, __fmul2_rn(dy, dy));
        const float2 q = __fmul2_rn(reach, reach);
        if (!(d2.x > q.x)) tcand |= 1u << (2 * mm);
        if (2 * mm + 1 < NMAX && !(d2.y > q.y)) tcand |= 1u << (2 * mm + 1);
      });
      tcand &= active;
    }
    if (tcand) {
      do {
        const int i = __ffs(tcand) - 1;
        tcand &= tcand - 1;
        const double xi = xl[i * kDB], yi = yl[i * kDB], ri = rl[i * kDB];
        const double dx = xi - tc.x, dy = yi - tc.y;
        const double reach = tr + ri;
        const double d2 = dx * dx + dy * dy;
        if (d2 > reach * reach) continue;  // the exact FP64 filter
        const double dist = sqrt(d2);
        const double depth = reach - dist;
        if (depth > 0.0) {
          double ux = 1.0, uy = 0.0;
          if (dist > 0.0) {
            const double inv = __drcp_rn(dist);  // == 1.0 / dist (both correctly rounded)
            ux = dx * inv;
            uy = dy * inv;
          }
          const double nx = xi + ux * depth, ny = yi + uy * depth;
          xl[i * kDB] = nx;
          yl[i * kDB] = ny;
          xs[i * kDB] = static_cast<float>(nx);
          ys[i * kDB] = static_cast<float>(ny);
          max_pen = dmax(max_pen, depth);
        }
      } while (tcand);
      static_for<NMAX>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        XF(i) = xs[i * kDB];
        YF(i) = ys[i * kDB];
      });
    }
    // 3-4. object pairs, lexicographic Gauss-Seidel (push_sim.cpp:101-117)
    // `near` = pairs within reach + kNear: a pair outside it cannot pass the
    // broad test until the objects have moved by kNear/2 in this pair sweep
    // (tracked in `swept`), so re-queues after a hit can skip it exactly.
    Mask<W> cand, near;
    cand.clear();
    near.clear();
    {
      // row i: pair (i, i+1) alone when i+1 is odd, then couples (j, j+1)
      // with j even, so {XF(j), XF(j+1)} is the stored float2
      const float2 m1 = make_float2(-1.f, -1.f);
      const float2 kn2 = make_float2(static_cast<float>(kNear), static_cast<float>(kNear));
      static_for<NMAX>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        constexpr int p0 = i * (2 * NMAX - i - 1) / 2;  // pair (i, i+1)
        const float2 xi2 = make_float2(XF(i), XF(i)), yi2 = make_float2(YF(i), YF(i));
        const float2 ri2 = make_float2(RM(i), RM(i));
        static_for<NMAX>([&](auto jc) {
          constexpr int j = decltype(jc)::value;
          constexpr int p = p0 + (j - i - 1);
          if constexpr (j > i && (j & 1) == 0 && j + 1 < NMAX) {
            const float2 dx = __ffma2_rn(xp[j >> 1], m1, xi2), dy = __ffma2_rn(yp[j >> 1], m1, yi2);
            const float2 rr = __fadd2_rn(ri2, rp[j >> 1]);
            const float2 d2 = __ffma2_rn(dx, dx, __fmul2_rn(dy, dy));
            const float2 q = __fmul2_rn(rr, rr);
            const float2 rn = __fadd2_rn(rr, kn2);
            const float2 qn = __fmul2_rn(rn, rn);
            if (!(d2.x > q.x)) cand.w[p >> 6] |= 1ull << (p & 63);
            if (!(d2.y > q.y)) cand.w[(p + 1) >> 6] |= 1ull << ((p + 1) & 63);
            if (!(d2.x > qn.x)) near.w[p >> 6] |= 1ull << (p & 63);
            if (!(d2.y > qn.y)) near.w[(p + 1) >> 6] |= 1ull << ((p + 1) & 63);
          } else if constexpr (j > i && ((j == i + 1 && (j & 1) == 1) || ((j & 1) == 0 && j + 1 == NMAX))) {
            const float dx = XF(i) - XF(j), dy = YF(i) - YF(j);
            const float rr = RM(i) + RM(j);
            const float d2 = __fmaf_rn(dx, dx, dy * dy);
            const float rn = rr + static_cast<float>(kNear);
            if (!(d2 > rr * rr)) cand.w[p >> 6] |= 1ull << (p & 63);
            if (!(d2 > rn * rn)) near.w[p >> 6] |= 1ull << (p & 63);
          }
        });
      });
    }
#pragma unroll
    for (int k = 0; k < W; ++k) {
      cand.w[k] &= pact.w[k];
      near.w[k] &= pact.w[k];
    }
    bool moved = false;
    double swept = 0.0;  // sum of the per-hit displacements in this sweep
    while (cand.any()) {
      const int p = cand.pop();
      const int ij = pij[p];
      const int i = ij & 0xff, j = ij >> 8;
      const double xi = xl[i * kDB], yi = yl[i * kDB], xj = xl[j * kDB], yj = yl[j * kDB];
      const double ri = rl[i * kDB], rj = rl[j * kDB];
      const double bx = xi - xj, by = yi - yj;
      const double rr = ri + rj;
      const double d2 = bx * bx + by * by;
      if (d2 > rr * rr) continue;  // stale candidate that no longer passes the broad test
      const double dx = xj - xi, dy = yj - yi;
      const double dist = sqrt(d2);  // norm2(pos_j - pos_i) == d2 bit for bit (negation is exact)
      const double depth = ri + rj - dist;
      if (depth > 0.0) {
        double ux = 1.0, uy = 0.0;
        if (dist > 0.0) {
          const double inv = __drcp_rn(dist);  // == 1.0 / dist (both correctly rounded)
          ux = dx * inv;
          uy = dy * inv;
        }
        const double s = 0.5 * depth;
        const double mx = ux * s, my = uy * s;
        const double nxi = xi - mx, nyi = yi - my, nxj = xj + mx, nyj = yj + my;
        xl[i * kDB] = nxi;
        yl[i * kDB] = nyi;
        xl[j * kDB] = nxj;
        yl[j * kDB] = nyj;
        xs[i * kDB] = static_cast<float>(nxi);
        ys[i * kDB] = static_cast<float>(nyi);
        xs[j * kDB] = static_cast<float>(nxj);
        ys[j * kDB] = static_cast<float>(nyj);
        max_pen = dmax(max_pen, depth);
        moved = true;
        // i and j moved: every LATER active pair touching them is re-queued
        // (re-tested when popped); other pairs' inputs are unchanged.  While
        // every object has moved less than kNear/2 since the broad pass (each
        // hit moves two objects by |u|*s <= s*(1+1e-15)), pairs outside
        // `near` still fail the broad test, so they are not re-queued.
        swept += s;
        cand.or_above(omask[i], omask[j], (2.0 * swept < kNear - 1e-9) ? near : pact, p);
      }
    }
    // 5. clamp every object (push_sim.cpp:118 -> :48-54).  clamp(v,-h,h) == v
    // whenever |v| <= h, so the clamp itself only runs for objects at a wall.
    // The float test is conservative (hclf = hcl - m); objects near a wall
    // take the exact path from shared memory.
    bool inside = true;
    static_for<NMAX>([&](auto ic) {
      constexpr int i = decltype(ic)::value;
      if (moved) {
        XF(i) = xs[i * kDB];
        YF(i) = ys[i * kDB];
      }
      inside = inside && fabsf(XF(i)) <= hclf && fabsf(YF(i)) <= hclf;
    });
    if (!inside) {
      for (int i = 0; i < n; ++i) {
        const double xi = xl[i * kDB], yi = yl[i * kDB];
        const double cx = fclampd(xi, -hcl, hcl), cy = fclampd(yi, -hcl, hcl);
        if (cx != xi || cy != yi) {
          xl[i * kDB] = cx;
          yl[i * kDB] = cy;
          xs[i * kDB] = static_cast<float>(cx);
          ys[i * kDB] = static_cast<float>(cy);
        }
      }
      static_for<NMAX>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        XF(i) = xs[i * kDB];
        YF(i) = ys[i * kDB];
      });
    }
    // Fixed point: the iteration left every position bit-identical, so each
    // remaining iteration of the substep repeats it exactly (max_pen > eps
    // each time) up to max_iters: the substep ends with this state.
    bool fixed = false;
    if (kFix && C.fixpoint && iter >= kFixK && !(max_pen <= C.eps_pen)) {
      fixed = true;
#pragma unroll 1
      for (int k = 0; k < n; ++k)
        fixed = fixed && __double_as_longlong(xl[k * kDB]) == __double_as_longlong(fx0[k]) &&
                __double_as_longlong(yl[k * kDB]) == __double_as_longlong(fy0[k]);
    }
    if (max_pen <= C.eps_pen || fixed || ++iter >= C.max_iters) {
      ++step;
      iter = 0;
    }
    if constexpr (kFix) {
      if (a.resume_si && --budget_left <= 0 && step <= C.substeps) {
        // wave rounds: yield — positions in place (discs do not rotate), progress saved
        double* out = a.poses_out + static_cast<size_t>(ee) * n * 3;
        for (int i = 0; i < n; ++i) {
          out[i * 3] = xl[i * kDB];
          out[i * 3 + 1] = yl[i * kDB];
        }
        a.resume_si[ee] = step << 8 | iter;
        a.resume_active[ee] = active;
        a.status[ee] = 3;
        e = atomicAdd(next_env, 1) + total_threads;
        need_init = true;
        have = false;
      }
    }
  }
#undef XF
#undef YF
#undef RM
}

#define PPG_DISC_INST(N)                                                                                       \
  template __global__ void resolve_disc_kernel<N, false>(const __grid_constant__ SimConst, ResolveArgs, int*); \
  template __global__ void resolve_disc_kernel<N, true>(const __grid_constant__ SimConst, ResolveArgs, int*);
PPG_DISC_INST(4)
PPG_DISC_INST(6)
PPG_DISC_INST(8)
PPG_DISC_INST(10)
PPG_DISC_INST(11)
PPG_DISC_INST(12)
PPG_DISC_INST(14)
PPG_DISC_INST(16)
PPG_DISC_INST(18)
PPG_DISC_INST(20)
#undef PPG_DISC_INST

}  // namespace ppg
