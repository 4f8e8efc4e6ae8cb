// dtree.cu — the device-resident PMBS search tree (north star
// item 3): batched UCT leaf selection with virtual loss, batched expansion,
// lockstep rollouts and batched backpropagation all run on the device, and
// ONE CUDA-graph launch executes one whole PMBS iteration (Algorithm 1 of
// arxiv 2207.06649; run_pmbs, pmbs.cpp:242-292).  The lockstep rounds run
// inside the graph under a conditional WHILE node whose condition the
// harvest kernel sets (n_active > 0), so the host only reads a few status
// words per iteration (stop flag, sizes) to decide whether to launch again.
//
// Decision-for-decision identical to the host planner (planner.cpp) and so
// to the reference:
//   select_batch / descend_virtual / ucb_virtual / pop_untried (pmbs.cpp:12-63,
//     mcts.cpp:13-16) -> dt_select_kernel: one block scores a node's
//     children in parallel, first maximum in insertion order; UCB with the host's glibc log
//     table and IEEE sqrt / division; subtree_selectable (pmbs.cpp:21-28) is
//     kept INCREMENTALLY as a per-node count of selectable children (selc)
//     instead of a recursive scan;
//   reset_virtual (pmbs.cpp:65-68) -> dt_gather_kernel;
//   batch_expand attach (pmbs.cpp:95-131, mcts.cpp:77-105) -> dt_attach_kernel
//     (child slot == popped untried index, so the batch-order append is a
//     parallel scatter) + dt_copy_kernel; d_T shrink (pmbs.cpp:119-127) and
//     update_es_level / level_settled (mcts.cpp:187-209) from per-level
//     counts of unsettled nodes;
//   batch_simulate (pmbs.cpp:207-234) -> the lockstep kernels with their
//     per-iteration values read on the device (LockArgs.dyn);
//   backprop_max -> backprop_mean (pmbs.cpp:236-240, mcts.cpp:180-185) ->
//     dt_backprop_kernel: lane d folds the rewards into the depth-d ancestor
//     in batch order (exact FP64 summation order);
//   early_stop_satisfied + budget (mcts.cpp:211-216, pmbs.cpp:282-290) ->
//     dt_stop_kernel.
// The final tree is read back once for best_root_child (mcts.cpp:218-235)
// and the tree signature (mcts.cpp:284-300).
#include <cuda_runtime.h>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>
#include <thread>
#include <vector>

#include "ctx_impl.cuh"

namespace ppg {

constexpr int kMaxTreeDepth = 32;
constexpr int kWideBackprop = 8192;  // batches from this size backprop regrouped by ancestor  // ancestor row stride; node depths <= tree_depth < 32

struct DTScal {
  int n_nodes;
  int n_pairs;          // this iteration's selections
  int dT, dS;           // tree_depth, rollout_depth
  int es_level;
  int min_grasp_depth;  // over attached graspable children (INT_MAX: none)
  int levels;           // max depth + 1
  int stop;             // -1 running, 0 budget, 1 explored, 2 early stop, 3 internal error
  int iteration;
  int recompute;        // d_T shrank this iteration: recount the selectable children
  int lock_dyn[6];      // LockArgs.dyn: n_nodes, used envs, depth cap, iteration, seed lo / hi
  int max_iters;        // iteration budget (0: seconds budget, checked by the host)
  double c_explore;     // UCB exploration constant
  // (the per-search values live here, not in the captured kernel arguments,
  // so one captured graph serves every search with the same shapes)
  long long a_used;     // action-pool entries in use
  long long expansions;
  int unsettled[kMaxTreeDepth];  // non-terminal nodes with untried actions, per depth
  int err[4];                    // first invariant violation seen on the device (debug)
  int round_mode;                // adaptive lockstep rounds (LockArgs.round_mode)
  int round_guard;               // rounds of this iteration's lockstep (< 0: limit hit)
  int async_ctl[16];             // asynchronous / wave lockstep control (LockArgs.a_ctl; [3] != 0: stalled)
};

struct DTree {
  // node arrays [cap_nodes]
  int32_t* parent;
  int32_t* depth;
  double* q;
  long long* visits;
  int32_t* vv;        // virtual visits
  uint8_t* flags;     // bit0 graspable, bit1 dead (terminal == flags != 0)
  long long* u_off;   // untried actions (apool) and children (cpool) share this offset
  int32_t* u_n;
  int32_t* u_head;
  int32_t* c_n;
  int32_t* selc;      // selectable children
  double* action;     // [cap][4]
  double* poses;      // [cap][n][3]
  int32_t* anc;       // [cap][kMaxTreeDepth]: ancestor at each depth (self at its own)
  double* apool;      // [cap_actions][4]
  int32_t* cpool;     // [cap_actions]
  // per-iteration batch [n_envs]
  int32_t* sel_node;
  long long* sel_act;
  double* gp;         // parent poses [P][n][3]
  double* ga;         // actions [P][4]
  double* cp;         // child poses [P][n][3] (the new nodes' poses, in batch order)
  int32_t* st;
  uint8_t* gr;
  int32_t* nu;
  double* un;         // [P][n*na][4]
  int32_t* meta;      // [P][3] depth, graspable, dead
  const unsigned long long* rew;  // lockstep per-new-node max reward bits
  const double* logtab;           // logtab[k] == glibc log((double)k)
  DTScal* sc;
  int n_envs, n, na, leaf_parallel;
};

namespace {

__device__ __forceinline__ bool dt_self(const DTree& t, int x, int dT) {
  return t.flags[x] == 0 && t.depth[x] < dT && t.u_head[x] < t.u_n[x];
}

// subtree_selectable (pmbs.cpp:21-28) under the selc invariant.
__device__ __forceinline__ bool dt_selectable(const DTree& t, int x, int dT) {
  return t.flags[x] == 0 && ((t.depth[x] < dT && t.u_head[x] < t.u_n[x]) || t.selc[x] > 0);
}

constexpr unsigned kAll = 0xffffffffu;

// select_batch (pmbs.cpp:52-63): up to n_envs descents with virtual visits,
// one block.  At every level the block scores the node's children in
// parallel (kSelThreads per round, loads of a round issued before scoring),
// reduces to the FIRST maximum in insertion order, and descends; thread 0
// pops the untried action and updates virtual visits / selectable counts.
constexpr int kSelThreads = 256;

// (score, insertion index, packed child) first-maximum merge; the packed
// child is 2 * node + dt_self(node), carried so the winner needs no reload.
__device__ __forceinline__ void sel_merge(double& bs, int& bk, int& bp, double os, int ok, int op) {
  if (os > bs || (os == bs && ok < bk)) {
    bs = os;
    bk = ok;
    bp = op;
  }
}

// Children of node x scored by the calling thread (children k = tid,
// tid + kSelThreads, ...; all loads of a chunk issued before any score):
// the thread's first maximum (score, insertion index, packed child).
__device__ __forceinline__ void dt_scan_children(const DTree& t, int x, double lg, int dT, double cexp, int tid,
                                                 double& bs, int& bk, int& bp) {
  const long long co = t.u_off[x];
  const int cn = t.c_n[x];
  constexpr int kScanU = 2;
  for (int k0 = 0; k0 < cn; k0 += kSelThreads * kScanU) {
    int ch[kScanU];
#pragma unroll
    for (int u = 0; u < kScanU; ++u) {
      const int k = k0 + kSelThreads * u + tid;
      ch[u] = k < cn ? t.cpool[co + k] : -1;
    }
    bool sel[kScanU], slf[kScanU];
    long long nci[kScanU];
    double qc[kScanU];
#pragma unroll
    for (int u = 0; u < kScanU; ++u) {
      const int c = ch[u] >= 0 ? ch[u] : 0;
      const bool ok = ch[u] >= 0 && t.flags[c] == 0;
      slf[u] = ok && t.depth[c] < dT && t.u_head[c] < t.u_n[c];
      sel[u] = slf[u] || (ok && t.selc[c] > 0);  // dt_selectable
      nci[u] = ch[u] >= 0 ? t.visits[c] + t.vv[c] : 0;
      qc[u] = ch[u] >= 0 ? t.q[c] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kScanU; ++u) {
      if (!sel[u]) continue;
      double sv = INFINITY;  // ucb_virtual (pmbs.cpp:12-17)
      if (nci[u] != 0) {
        const double nc = static_cast<double>(nci[u]);
        sv = qc[u] / nc + cexp * sqrt(2.0 * lg / nc);
      }
      if (sv > bs) {
        bs = sv;
        bk = k0 + kSelThreads * u + tid;
        bp = 2 * ch[u] + (slf[u] ? 1 : 0);
      }
    }
  }
}

// Block-wide first maximum of the threads' (score, index, packed child):
// warp reduction, per-warp partials (double-buffered by `parity`, ONE block
// barrier), then every warp reduces the partials itself.
template <int kWarps>
__device__ __forceinline__ void dt_block_best(double& bs, int& bk, int& bp, double (*s_bs)[kWarps],
                                              int (*s_bk)[kWarps], int (*s_bp)[kWarps], int& parity, int l,
                                              int wid) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)  // first maximum in insertion order
    sel_merge(bs, bk, bp, __shfl_xor_sync(kAll, bs, o), __shfl_xor_sync(kAll, bk, o), __shfl_xor_sync(kAll, bp, o));
  if (l == 0) {
    s_bs[parity][wid] = bs;
    s_bk[parity][wid] = bk;
    s_bp[parity][wid] = bp;
  }
  __syncthreads();
  bs = l < kWarps ? s_bs[parity][l] : -INFINITY;
  bk = l < kWarps ? s_bk[parity][l] : INT_MAX;
  bp = l < kWarps ? s_bp[parity][l] : -2;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
    sel_merge(bs, bk, bp, __shfl_xor_sync(kAll, bs, o), __shfl_xor_sync(kAll, bk, o), __shfl_xor_sync(kAll, bp, o));
  parity ^= 1;
}

// The root and its children are the nodes every draw reads and updates
// (virtual visits, untried heads, selectable counts): with up to
// kSelCache children they live in shared memory for the whole kernel and are
// written back at the end; deeper levels read the tree in HBM.
constexpr int kSelCache = 512;

__global__ void __launch_bounds__(kSelThreads) dt_select_kernel(DTree t) {
  constexpr int kWarps = kSelThreads / 32;
  __shared__ double s_bs[2][kWarps];
  __shared__ int s_bk[2][kWarps], s_bp[2][kWarps];
  // root-children cache (slot k = insertion index k of the root's children)
  __shared__ int s_ch[kSelCache], s_vv[kSelCache], s_uh[kSelCache], s_un[kSelCache], s_selc[kSelCache],
      s_dep[kSelCache];
  __shared__ long long s_vis[kSelCache];
  __shared__ double s_q[kSelCache];
  __shared__ uint8_t s_fl[kSelCache];
  __shared__ long long s_rvis;
  __shared__ int s_r[6];  // root: vv, u_head, u_n, selc, flags, depth
  DTScal* sc = t.sc;
  const int tid = threadIdx.x, l = tid & 31, wid = tid >> 5;
  const int dT = sc->dT;
  const double cexp = sc->c_explore;
  int draws = 0;
  bool bad = false;
  int parity = 0;
  const int cn0 = t.c_n[0];
  const bool cached = cn0 <= kSelCache;
  if (sc->stop < 0 && cached) {
    const long long co0 = t.u_off[0];
    for (int k = tid; k < cn0; k += kSelThreads) {
      const int c = t.cpool[co0 + k];
      s_ch[k] = c;
      s_vv[k] = t.vv[c];
      s_uh[k] = t.u_head[c];
      s_un[k] = t.u_n[c];
      s_selc[k] = t.selc[c];
      s_dep[k] = t.depth[c];
      s_vis[k] = t.visits[c];
      s_q[k] = t.q[c];
      s_fl[k] = t.flags[c];
    }
    if (tid == 0) {
      s_rvis = t.visits[0];
      s_r[0] = t.vv[0];
      s_r[1] = t.u_head[0];
      s_r[2] = t.u_n[0];
      s_r[3] = t.selc[0];
      s_r[4] = t.flags[0];
      s_r[5] = t.depth[0];
    }
    __syncthreads();
    for (; draws < t.n_envs; ++draws) {
      // subtree_selectable(root) / is the root itself expandable
      const bool rself = s_r[4] == 0 && s_r[5] < dT && s_r[1] < s_r[2];
      if (!(rself || (s_r[4] == 0 && s_r[3] > 0))) break;
      int x = 0, lvl = 0, slot1 = -1;
      int my_node = 0;  // thread d keeps the root path's node at depth d
      bool self = rself;
      if (!self) {  // descend_virtual (pmbs.cpp:30-48), the root level from the cache
        const double lg = t.logtab[s_rvis + s_r[0]];
        double bs = -INFINITY;
        int bk = INT_MAX, bp = -2;
        for (int k = tid; k < cn0; k += kSelThreads) {
          const bool ok = s_fl[k] == 0;
          const bool slf = ok && s_dep[k] < dT && s_uh[k] < s_un[k];
          if (!(slf || (ok && s_selc[k] > 0))) continue;
          const long long nci = s_vis[k] + s_vv[k];
          double sv = INFINITY;  // ucb_virtual (pmbs.cpp:12-17)
          if (nci != 0) {
            const double nc = static_cast<double>(nci);
            sv = s_q[k] / nc + cexp * sqrt(2.0 * lg / nc);
          }
          if (sv > bs) {
            bs = sv;
            bk = k;
            bp = 2 * s_ch[k] + (slf ? 1 : 0);
          }
        }
        dt_block_best<kWarps>(bs, bk, bp, s_bs, s_bk, s_bp, parity, l, wid);
        ++lvl;
        if (bk == INT_MAX) {
          bad = true;
        } else {
          x = bp >> 1;
          self = (bp & 1) != 0;
          slot1 = bk;
          if (tid == 1) my_node = x;
        }
        while (!bad && !self) {  // deeper levels from HBM
          const int vx = lvl == 1 ? s_vv[slot1] : t.vv[x];
          const double lgx = t.logtab[t.visits[x] + vx];
          bs = -INFINITY;
          bk = INT_MAX;
          bp = -2;
          dt_scan_children(t, x, lgx, dT, cexp, tid, bs, bk, bp);
          dt_block_best<kWarps>(bs, bk, bp, s_bs, s_bk, s_bp, parity, l, wid);
          ++lvl;
          if (bk == INT_MAX) {  // impossible under the selc invariant
            bad = true;
            break;
          }
          x = bp >> 1;
          self = (bp & 1) != 0;
          if (tid == lvl) my_node = x;
        }
      }
      if (bad) break;
      // virtual visit on the root path (one node per thread)
      if (tid == 0) s_r[0] += 1;
      else if (tid == 1 && lvl >= 1) s_vv[slot1] += 1;
      else if (tid <= lvl) t.vv[my_node] += 1;
      if (tid == 0) {  // pop_untried (mcts.cpp:13-16)
        int h, un, dx;
        if (lvl == 0) {
          h = s_r[1]++;
          un = s_r[2];
          dx = s_r[5];
        } else if (lvl == 1) {
          h = s_uh[slot1]++;
          un = s_un[slot1];
          dx = s_dep[slot1];
        } else {
          h = t.u_head[x];
          t.u_head[x] = h + 1;
          un = t.u_n[x];
          dx = t.depth[x];
        }
        t.sel_node[draws] = x;
        t.sel_act[draws] = t.u_off[x] + h;
        if (h + 1 == un) {  // now fully expanded
          sc->unsettled[dx] -= 1;
          const int sx = lvl == 0 ? s_r[3] : lvl == 1 ? s_selc[slot1] : t.selc[x];
          if (sx == 0) {  // x left the selectable set: update its ancestors (all on this draw's path)
            for (int d = lvl - 1; d >= 0; --d) {
              bool still;
              if (d == 0) {
                s_r[3] -= 1;
                still = s_r[4] == 0 && ((s_r[5] < dT && s_r[1] < s_r[2]) || s_r[3] > 0);
              } else if (d == 1) {
                s_selc[slot1] -= 1;
                still = s_fl[slot1] == 0 && ((s_dep[slot1] < dT && s_uh[slot1] < s_un[slot1]) || s_selc[slot1] > 0);
              } else {
                // the ancestor at depth d: walk up from x
                int p = x;
                for (int k = lvl; k > d; --k) p = t.parent[p];
                t.selc[p] -= 1;
                still = dt_selectable(t, p, dT);
              }
              if (still) break;
            }
          }
        }
      }
      __syncthreads();
    }
    // write the cached nodes back
    if (tid == 0) {
      t.vv[0] = s_r[0];
      t.u_head[0] = s_r[1];
      t.selc[0] = s_r[3];
    }
    for (int k = tid; k < cn0; k += kSelThreads) {
      const int c = s_ch[k];
      t.vv[c] = s_vv[k];
      t.u_head[c] = s_uh[k];
      t.selc[c] = s_selc[k];
    }
  } else if (sc->stop < 0) {
    for (; draws < t.n_envs; ++draws) {
      if (!dt_selectable(t, 0, dT)) break;  // every thread reads the same state
      int x = 0, lvl = 0;
      int my_node = 0;
      bool self = dt_self(t, 0, dT);
      while (!self) {  // descend_virtual (pmbs.cpp:30-48)
        const double lg = t.logtab[t.visits[x] + t.vv[x]];  // log(n_parent)
        double bs = -INFINITY;
        int bk = INT_MAX, bp = -2;
        dt_scan_children(t, x, lg, dT, cexp, tid, bs, bk, bp);
        dt_block_best<kWarps>(bs, bk, bp, s_bs, s_bk, s_bp, parity, l, wid);
        ++lvl;
        if (bk == INT_MAX) {  // impossible under the selc invariant
          bad = true;
          break;
        }
        x = bp >> 1;
        self = (bp & 1) != 0;
        if (tid == lvl) my_node = x;
      }
      if (bad) break;
      if (tid <= lvl) t.vv[my_node] += 1;  // virtual visit on the root path (one node per thread)
      if (tid == 0) {  // pop_untried (mcts.cpp:13-16)
        const int h = t.u_head[x];
        t.sel_node[draws] = x;
        t.sel_act[draws] = t.u_off[x] + h;
        t.u_head[x] = h + 1;
        if (h + 1 == t.u_n[x]) {  // now fully expanded
          sc->unsettled[t.depth[x]] -= 1;
          if (t.selc[x] == 0)  // x left the selectable set: update its ancestors
            for (int p = t.parent[x]; p >= 0; p = t.parent[p]) {
              t.selc[p] -= 1;
              if (dt_selectable(t, p, dT)) break;
            }
        }
      }
      __syncthreads();
    }
  }
  if (tid == 0) {
    sc->n_pairs = draws;
    if (bad) sc->stop = 3;
    else if (draws == 0 && sc->stop < 0) sc->stop = 1;  // TreeExhausted: explored
  }
}

// The root node + the search scalars from one staged block (dt_begin):
// [DTScal][root flags (int)][root poses n*3 doubles].
__global__ void dt_root_kernel(DTree t, const char* stage, int n, int cnt, long long* counters) {
  const int tid = threadIdx.x;
  const DTScal* h = reinterpret_cast<const DTScal*>(stage);
  const int rf = *reinterpret_cast<const int*>(stage + sizeof(DTScal));
  const double* rp = reinterpret_cast<const double*>(stage + sizeof(DTScal) + 8);
  if (tid == 0) {
    t.parent[0] = -1;
    t.depth[0] = 0;
    t.q[0] = 0.0;
    t.visits[0] = 0;
    t.vv[0] = 0;
    t.flags[0] = static_cast<uint8_t>(rf);
    t.u_off[0] = 0;
    t.u_n[0] = cnt;
    t.u_head[0] = 0;
    t.c_n[0] = 0;
    t.selc[0] = 0;
    t.anc[0] = 0;
  }
  if (tid < 4) t.action[tid] = 0.0;
  if (tid < 4) counters[tid] = 0;
  for (int i = tid; i < n * 3; i += blockDim.x) t.poses[i] = rp[i];
  const int* src = reinterpret_cast<const int*>(h);
  int* dst = reinterpret_cast<int*>(t.sc);
  for (int i = tid; i < static_cast<int>(sizeof(DTScal) / 4); i += blockDim.x) dst[i] = src[i];
}

// The final read-back's children lists, dense: node x's children at
// kids[coff[x] .. coff[x] + c_n[x]) (coff = exclusive scan of c_n), instead
// of the whole action-sized children pool.
__global__ void dt_kids_kernel(DTree t, int N, const int* coff, int* kids) {
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < N; x += gridDim.x * blockDim.x) {
    const long long o = t.u_off[x];
    const int b = coff[x], m = t.c_n[x];
    for (int k = 0; k < m; ++k) kids[b + k] = t.cpool[o + k];
  }
}

// reset_virtual (pmbs.cpp:65-68) + gather of the batch's parent poses and
// actions (and the child-pose buffer the in-place disc kernel resolves).
__global__ void dt_gather_kernel(DTree t, bool copy_child) {
  const int P = t.sc->n_pairs, N = t.sc->n_nodes, n3 = t.n * 3;
  const int g = blockIdx.x * blockDim.x + threadIdx.x, G = gridDim.x * blockDim.x;
  for (int i = g; i < N; i += G) t.vv[i] = 0;
  for (int i = g; i < P * n3; i += G) {
    const int k = i / n3, r = i - k * n3;
    const double v = t.poses[static_cast<size_t>(t.sel_node[k]) * n3 + r];
    t.gp[i] = v;
    if (copy_child) t.cp[i] = v;
  }
  for (int i = g; i < P * 4; i += G) t.ga[i] = t.apool[t.sel_act[i >> 2] * 4 + (i & 3)];
}

// batch_expand attach (pmbs.cpp:95-131) for the whole batch at once.  One
// block.  Every pop produced exactly one child, so the child created from
// untried index h of node p sits in children slot h: the batch-order append
// is a scatter.  Untried lists are appended to the pool in batch order (block
// scan).  Selectable-children counts are updated with atomics ("first
// incrementer propagates"); if d_T shrinks they are recounted instead.
__global__ void __launch_bounds__(1024) dt_attach_kernel(DTree t) {
  DTScal* sc = t.sc;
  const int P = sc->n_pairs;
  const int tid = threadIdx.x, B = blockDim.x;
  __shared__ long long s_part[1024];
  __shared__ int s_mind, s_maxd;
  if (P == 0) {
    if (tid == 0) {
      sc->lock_dyn[0] = 0;
      sc->lock_dyn[1] = 0;
      sc->lock_dyn[2] = sc->dT + sc->dS;
      sc->lock_dyn[3] = sc->iteration;
    }
    return;
  }
  const int base = sc->n_nodes, dT0 = sc->dT;
  const long long a0 = sc->a_used;
  if (tid == 0) {
    s_mind = INT_MAX;
    s_maxd = 0;
  }
  // exclusive scan of the untried counts of the live children, batch order
  const int chunk = (P + B - 1) / B;
  const int k0 = tid * chunk, k1 = min(P, k0 + chunk);
  long long loc = 0;
  for (int k = k0; k < k1; ++k) loc += t.st[k] == 0 ? t.nu[k] : 0;
  s_part[tid] = loc;
  __syncthreads();
  for (int off = 1; off < B; off <<= 1) {  // Hillis-Steele inclusive scan
    const long long v = tid >= off ? s_part[tid - off] : 0;
    __syncthreads();
    s_part[tid] += v;
    __syncthreads();
  }
  long long run = a0 + s_part[tid] - loc;
  for (int k = k0; k < k1; ++k) {
    const int id = base + k, p = t.sel_node[k], d = t.depth[p] + 1;
    const bool alive = t.st[k] == 0;  // a failed simulation yields a dead child (pmbs.cpp:105-107)
    const bool g = alive && t.gr[k] != 0;
    const int un = alive ? t.nu[k] : 0;
    const bool dead = !g && un == 0;
    t.parent[id] = p;
    t.depth[id] = d;
    t.q[id] = 0.0;
    t.visits[id] = 0;
    t.vv[id] = 0;
    t.flags[id] = static_cast<uint8_t>((g ? 1 : 0) | (dead ? 2 : 0));
    t.u_off[id] = run;
    run += un;
    t.u_n[id] = un;
    t.u_head[id] = 0;
    t.c_n[id] = 0;
    t.selc[id] = 0;
    const long long h = t.sel_act[k] - t.u_off[p];
    t.cpool[t.u_off[p] + h] = id;
    t.c_n[p] = t.u_head[p];  // every pop so far has its child now (same value from every writer)
    t.meta[k * 3] = d;
    t.meta[k * 3 + 1] = g ? 1 : 0;
    t.meta[k * 3 + 2] = dead ? 1 : 0;
    if (!g && !dead) atomicAdd(&sc->unsettled[d], 1);  // non-terminal with untried actions
    if (g) atomicMin(&s_mind, d);
    atomicMax(&s_maxd, d);
    if (!g && !dead && d < dT0) {  // a selectable child: p (and maybe ancestors) become selectable
      for (int x = p; x >= 0; x = t.parent[x]) {
        const int old = atomicAdd(&t.selc[x], 1);
        if (old > 0 || dt_self(t, x, dT0)) break;
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    sc->n_nodes = base + P;
    sc->a_used = a0 + s_part[B - 1];
    sc->levels = max(sc->levels, s_maxd + 1);
    sc->recompute = 0;
    if (s_mind < INT_MAX) {
      sc->min_grasp_depth = min(sc->min_grasp_depth, s_mind);
      if (s_mind < sc->dT) {  // shallower graspable child (pmbs.cpp:119-127)
        sc->dT = s_mind;
        sc->dS = 0;
        sc->recompute = 1;
      }
    }
    // update_es_level (mcts.cpp:202-209) with level_settled (:189-198)
    if (sc->es_level <= sc->dT) {
      const int L = sc->es_level - 1;
      const bool settled = L < 0 || L >= sc->levels || L >= sc->dT || sc->unsettled[L] == 0;
      if (settled) sc->es_level += 1;
    }
    sc->lock_dyn[0] = P;
    sc->lock_dyn[1] = t.leaf_parallel ? t.n_envs : P;
    sc->lock_dyn[2] = sc->dT + sc->dS;
    sc->lock_dyn[3] = sc->iteration;
  }
}

// Recount selc bottom-up after d_T shrank (selectability of every node may
// have changed).  One block, one pass per depth level.
__global__ void __launch_bounds__(1024) dt_recount_kernel(DTree t) {
  const DTScal* sc = t.sc;
  if (!sc->recompute) return;
  const int N = sc->n_nodes, dT = sc->dT;
  for (int L = sc->levels - 1; L >= 0; --L) {
    for (int x = threadIdx.x; x < N; x += blockDim.x) {
      if (t.depth[x] != L) continue;
      int c = 0;
      const long long co = t.u_off[x];
      for (int k = 0; k < t.c_n[x]; ++k) c += dt_selectable(t, t.cpool[co + k], dT) ? 1 : 0;
      t.selc[x] = c;
    }
    __syncthreads();
  }
}

// The new nodes' poses, actions, untried lists and ancestor rows.
__global__ void dt_copy_kernel(DTree t) {
  const DTScal* sc = t.sc;
  const int P = sc->n_pairs, base = sc->n_nodes - P, n3 = t.n * 3, cap = t.n * t.na * 4;
  const int g = blockIdx.x * blockDim.x + threadIdx.x, G = gridDim.x * blockDim.x;
  for (int i = g; i < P * n3; i += G) t.poses[static_cast<size_t>(base) * n3 + i] = t.cp[i];
  for (int i = g; i < P * 4; i += G) t.action[static_cast<size_t>(base) * 4 + i] = t.ga[i];
  for (int i = g; i < P * kMaxTreeDepth; i += G) {
    const int k = i / kMaxTreeDepth, d = i - k * kMaxTreeDepth, id = base + k;
    const int dd = t.depth[id];
    if (d < dd) t.anc[static_cast<size_t>(id) * kMaxTreeDepth + d] = t.anc[static_cast<size_t>(t.sel_node[k]) * kMaxTreeDepth + d];
    else if (d == dd) t.anc[static_cast<size_t>(id) * kMaxTreeDepth + d] = id;
  }
  for (int k = blockIdx.x; k < P; k += gridDim.x) {
    const int id = base + k, un = t.u_n[id];
    const double* src = t.un + static_cast<size_t>(k) * cap;
    double* dst = t.apool + t.u_off[id] * 4;
    for (int i = threadIdx.x; i < un * 4; i += blockDim.x) dst[i] = src[i];
  }
}

// backprop_max -> backprop_mean (pmbs.cpp:236-240, mcts.cpp:180-185): for
// each new node in batch order, q_sum += r and visits += 1 on every node of
// its root path.  Lane d owns depth d, so each node's additions happen in
// batch order (the FP64 sum is the reference's).
__global__ void __launch_bounds__(32) dt_backprop_kernel(DTree t) {
  const DTScal* sc = t.sc;
  const int P = sc->n_pairs, base = sc->n_nodes - P, d = threadIdx.x;
  int cur = -1;
  double cq = 0.0;
  long long cv = 0;
  // 32 new nodes at a time: lane j fetches node k0 + j's depth and reward,
  // every lane fetches its depth's ancestor of all 32 (independent loads),
  // then the batch-order fold runs on shuffled values
  for (int k0 = 0; k0 < P; k0 += 32) {
    const int kj = k0 + d;
    const int Dj = kj < P ? t.depth[base + kj] : -1;
    const double rj = kj < P ? __longlong_as_double(static_cast<long long>(t.rew[kj])) : 0.0;
    int anc[32];
#pragma unroll
    for (int j = 0; j < 32; ++j)
      anc[j] = k0 + j < P ? t.anc[static_cast<size_t>(base + k0 + j) * kMaxTreeDepth + d] : -1;
    const int m = P - k0 < 32 ? P - k0 : 32;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      if (j >= m) break;
      const int id = base + k0 + j;
      const int D = __shfl_sync(kAll, Dj, j);
      const double r = __shfl_sync(kAll, rj, j);
      if (d == D) {
        t.q[id] = 0.0 + r;
        t.visits[id] = 1;
      } else if (d < D) {
        const int a = anc[j];
        if (a < 0 || a >= sc->n_nodes) {  // corrupt ancestor row: report, do not touch memory
          if (atomicCAS(const_cast<int*>(&sc->err[0]), 0, 1) == 0) {
            const_cast<DTScal*>(sc)->err[1] = id;
            const_cast<DTScal*>(sc)->err[2] = d;
            const_cast<DTScal*>(sc)->err[3] = a;
          }
          continue;
        }
        if (a != cur) {
          if (cur >= 0) {
            t.q[cur] = cq;
            t.visits[cur] = cv;
          }
          cur = a;
          cq = t.q[a];
          cv = t.visits[a];
        }
        cq += r;
        cv += 1;
      }
    }
  }
  if (cur >= 0) {
    t.q[cur] = cq;
    t.visits[cur] = cv;
  }
}

// Wide batches: the same backprop with the pairs regrouped by ancestor.
// Entry (p, d) = (ancestor of new node p at depth d, p); a stable sort by
// ancestor keeps each ancestor's pairs in batch order, and one thread folds
// each ancestor's rewards in that order — the FP64 sums of the sequential
// fold, without 32 lanes stepping through every pair.
__global__ void dt_bp_keys_kernel(DTree t, int dmax, int* keys, int* vals) {
  const DTScal* sc = t.sc;
  const int P = sc->n_pairs, N = sc->n_nodes, base = N - P;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int E = t.n_envs;
  if (i >= E * dmax) return;
  const int p = i / dmax, d = i - p * dmax;
  int key = INT_MAX;
  if (p < P) {
    const int id = base + p;
    const int D = t.depth[id];
    if (d == 0) {  // the new node itself
      t.q[id] = 0.0 + __longlong_as_double(static_cast<long long>(t.rew[p]));
      t.visits[id] = 1;
    }
    if (d < D) {
      const int a = t.anc[static_cast<size_t>(id) * kMaxTreeDepth + d];
      if (a < 0 || a >= N) {  // corrupt ancestor row: report, do not touch memory
        if (atomicCAS(const_cast<int*>(&sc->err[0]), 0, 1) == 0) {
          const_cast<DTScal*>(sc)->err[1] = id;
          const_cast<DTScal*>(sc)->err[2] = d;
          const_cast<DTScal*>(sc)->err[3] = a;
        }
      } else {
        key = a;
      }
    }
  }
  keys[i] = key;
  vals[i] = p;
}

__global__ void dt_bp_fold_kernel(DTree t, const int* keys, const int* vals, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int a = keys[i];
  if (a == INT_MAX || (i > 0 && keys[i - 1] == a)) return;  // not the head of an ancestor's run
  double cq = t.q[a];
  long long cv = t.visits[a];
  for (int j = i; j < n && keys[j] == a; ++j) {
    cq += __longlong_as_double(static_cast<long long>(t.rew[vals[j]]));
    cv += 1;
  }
  t.q[a] = cq;
  t.visits[a] = cv;
}

// End of an iteration: early stop (mcts.cpp:211-216) then the iteration
// budget (pmbs.cpp:282-290).
__global__ void dt_stop_kernel(DTree t) {
  DTScal* sc = t.sc;
  const int P = sc->n_pairs;
  if (P == 0) return;
  sc->iteration += 1;
  sc->expansions += P;
  if (sc->stop >= 0) return;
  if (sc->min_grasp_depth <= sc->es_level) sc->stop = 2;
  else if (sc->max_iters > 0 && sc->iteration >= sc->max_iters) sc->stop = 0;
}

}  // namespace

// ---------------------------------------------------------------------------
// host side

struct DTreeState {
  // tree
  DevBuf parent, depth, q, visits, vv, flags, u_off, u_n, u_head, c_n, selc, action, poses, anc, apool, cpool;
  // batch
  DevBuf sel_node, sel_act, gp, ga, cp, st, gr, nu, un, meta, logtab, sc;
  // lockstep state
  DevBuf l_node, l_pushes, l_done, l_byg, l_harv, l_flag, l_reward, l_poses, l_mt, l_mtidx, l_W, l_rew, l_active,
      l_nactive, l_counters, l_push, l_status, l_stepping, l_around, l_astate, l_aW, l_actr, l_adl, l_fin, l_rsi,
      l_ract, l_aP, l_spec;
  int cap_nodes = 0;
  long long cap_actions = 0;
  int n_envs = 0, n = 0, na = 0;
  cudaGraphExec_t exec = nullptr;  // the iteration (or its pre part when hooked)
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec_post = nullptr;  // hooked / sharded: backprop + stop
  cudaGraph_t graph_post = nullptr;
  cudaGraphExec_t exec_round = nullptr;  // sharded: one lockstep round + the local harvest half
  cudaGraph_t graph_round = nullptr;
  cudaStream_t st2 = nullptr;
  DTree t{};
  LockArgs la{};
  ResolveArgs lra{};
  SimConst C{};
  std::string key;  // configuration the graph was captured for
  // pinned host staging: the search start's root block, the per-iteration
  // scalars and the final tree read-back (one async copy each, no pageable
  // round trips)
  char* hpin = nullptr;
  size_t hpin_cap = 0;
  DTScal* hsc = nullptr;  // pinned copy of the scalars, read after every iteration
  DevBuf dstage;
  DevBuf bp_buf;  // wide-batch backprop: keys / values (x2) + sort scratch
  char* pinned(size_t bytes) {
    if (bytes > hpin_cap) {
      if (hpin) cudaFreeHost(hpin);
      hpin = nullptr;
      hpin_cap = 0;
      const size_t want = bytes < 4096 ? 4096 : bytes + bytes / 2;
      if (cudaMallocHost(&hpin, want) != cudaSuccess) return nullptr;
      hpin_cap = want;
    }
    return hpin;
  }
  // the last finished search (ppg_tree_export)
  bool last_valid = false;
  int last_nodes = 0, last_dT = 0, last_dS = 0, last_es = 0;
  long long last_a_used = 0;

  void release_graph() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    if (exec_post) cudaGraphExecDestroy(exec_post);
    if (graph_post) cudaGraphDestroy(graph_post);
    if (exec_round) cudaGraphExecDestroy(exec_round);
    if (graph_round) cudaGraphDestroy(graph_round);
    exec = exec_post = exec_round = nullptr;
    graph = graph_post = graph_round = nullptr;
  }
  void release() {
    release_graph();
    if (st2) cudaStreamDestroy(st2);
    st2 = nullptr;
    if (hpin) cudaFreeHost(hpin);
    hpin = nullptr;
    hpin_cap = 0;
    if (hsc) cudaFreeHost(hsc);
    hsc = nullptr;
    dstage.release();
    bp_buf.release();
    DevBuf* bufs[] = {&parent, &depth, &q, &visits, &vv, &flags, &u_off, &u_n, &u_head, &c_n, &selc, &action,
                      &poses, &anc, &apool, &cpool, &sel_node, &sel_act, &gp, &ga, &cp, &st, &gr, &nu, &un,
                      &meta, &logtab, &sc, &l_node, &l_pushes, &l_done, &l_byg, &l_harv, &l_flag, &l_reward,
                      &l_poses, &l_mt, &l_mtidx, &l_W, &l_rew, &l_active, &l_nactive, &l_counters, &l_push,
                      &l_status, &l_stepping, &l_around, &l_astate, &l_aW, &l_actr, &l_adl, &l_fin, &l_rsi, &l_ract, &l_aP,
                      &l_spec};
    for (DevBuf* b : bufs) b->release();
  }
};

void dtree_release(ppg_ctx* ctx) {
  if (ctx->dtree) {
    ctx->dtree->release();
    delete ctx->dtree;
    ctx->dtree = nullptr;
  }
}

namespace {

// Grows a node- or action-indexed buffer to `want` elements of `esz` bytes,
// preserving the first `used` elements.
cudaError_t grow(DevBuf& b, size_t want, size_t used, size_t esz, cudaStream_t st) {
  if (want * esz <= b.cap) return cudaSuccess;
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, want * esz);
  if (e != cudaSuccess) return e;
  if (b.p && used) e = cudaMemcpyAsync(p, b.p, used * esz, cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return e;
  if (b.p) {
    cudaStreamSynchronize(st);
    cudaFree(b.p);
  }
  b.p = p;
  b.cap = want * esz;
  return cudaSuccess;
}

double ucb_score_host(double q, long vis_child, long vis_parent, double c) {  // mcts.cpp:41-46
  if (vis_child == 0) return std::numeric_limits<double>::infinity();
  const double mean = q / static_cast<double>(vis_child);
  return mean + c * std::sqrt(2.0 * std::log(static_cast<double>(vis_parent)) / static_cast<double>(vis_child));
}

uint64_t fnv1a(const std::string& s) {
  uint64_t h = 1469598103934665603ull;
  for (unsigned char ch : s) {
    h ^= ch;
    h *= 1099511628211ull;
  }
  return h;
}

}  // namespace

}  // namespace ppg

using namespace ppg;

#define DCK(call)                                                                        \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess) {                                                             \
      ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);                     \
      return PPG_ECUDA;                                                                  \
    }                                                                                    \
  } while (0)

namespace {

// Ensures tree capacity for `nodes` nodes and `actions` pool entries.
int dt_reserve(ppg_ctx* ctx, DTreeState& S, int used_nodes, long long used_actions, int nodes, long long actions) {
  cudaStream_t st = ctx->stream;
  const int n = S.n;
  if (nodes > S.cap_nodes) {
    const size_t want = static_cast<size_t>(nodes), u = static_cast<size_t>(used_nodes);
    DCK(grow(S.parent, want, u, 4, st));
    DCK(grow(S.depth, want, u, 4, st));
    DCK(grow(S.q, want, u, 8, st));
    DCK(grow(S.visits, want, u, 8, st));
    DCK(grow(S.vv, want, u, 4, st));
    DCK(grow(S.flags, want, u, 1, st));
    DCK(grow(S.u_off, want, u, 8, st));
    DCK(grow(S.u_n, want, u, 4, st));
    DCK(grow(S.u_head, want, u, 4, st));
    DCK(grow(S.c_n, want, u, 4, st));
    DCK(grow(S.selc, want, u, 4, st));
    DCK(grow(S.action, want, u, 32, st));
    DCK(grow(S.poses, want, u, static_cast<size_t>(n) * 24, st));
    DCK(grow(S.anc, want, u, kMaxTreeDepth * 4, st));
    // log table: index visits + virtual visits <= nodes + n_envs
    const size_t lt = want + static_cast<size_t>(S.n_envs) + 2;
    std::vector<double> tab(lt);
    for (size_t k = 0; k < lt; ++k) tab[k] = std::log(static_cast<double>(k));
    DCK(S.logtab.ensure(lt * 8));
    DCK(cudaMemcpyAsync(S.logtab.p, tab.data(), lt * 8, cudaMemcpyHostToDevice, st));
    DCK(cudaStreamSynchronize(st));
    S.cap_nodes = nodes;
    S.release_graph();
  }
  if (actions > S.cap_actions) {
    DCK(grow(S.apool, static_cast<size_t>(actions), static_cast<size_t>(used_actions), 32, st));
    DCK(grow(S.cpool, static_cast<size_t>(actions), static_cast<size_t>(used_actions), 4, st));
    S.cap_actions = actions;
    S.release_graph();
  }
  return PPG_SUCCESS;
}

// Per-search batch + lockstep buffers (sized by n_envs).
int dt_batch(ppg_ctx* ctx, DTreeState& S) {
  const int E = S.n_envs, n = S.n, na = S.na;
  DCK(S.sel_node.ensure(static_cast<size_t>(E) * 4));
  DCK(S.sel_act.ensure(static_cast<size_t>(E) * 8));
  DCK(S.gp.ensure(static_cast<size_t>(E) * n * 24));
  DCK(S.ga.ensure(static_cast<size_t>(E) * 32));
  DCK(S.cp.ensure(static_cast<size_t>(E) * n * 24));
  DCK(S.st.ensure(static_cast<size_t>(E) * 4));
  DCK(S.gr.ensure(static_cast<size_t>(E)));
  DCK(S.nu.ensure(static_cast<size_t>(E) * 4));
  DCK(S.un.ensure(static_cast<size_t>(E) * n * na * 32));
  DCK(S.meta.ensure(static_cast<size_t>(E) * 12));
  DCK(S.sc.ensure(sizeof(DTScal)));
  DCK(S.l_node.ensure(static_cast<size_t>(E) * 4));
  DCK(S.l_pushes.ensure(static_cast<size_t>(E) * 4));
  DCK(S.l_done.ensure(E));
  DCK(S.l_byg.ensure(E));
  DCK(S.l_harv.ensure(E));
  DCK(S.l_flag.ensure(E));
  DCK(S.l_reward.ensure(static_cast<size_t>(E) * 8));
  DCK(S.l_poses.ensure(static_cast<size_t>(E) * n * 24));
  DCK(S.l_mt.ensure(static_cast<size_t>(E) * 312 * 8));
  DCK(S.l_mtidx.ensure(static_cast<size_t>(E) * 4));
  DCK(S.l_W.ensure(static_cast<size_t>(E) * 4));
  DCK(S.l_rew.ensure(static_cast<size_t>(E) * 8));
  DCK(S.l_active.ensure(static_cast<size_t>(E) * 4));
  DCK(S.l_nactive.ensure(16));
  DCK(S.l_counters.ensure(32));
  DCK(S.l_push.ensure(static_cast<size_t>(E) * 32));
  DCK(S.l_status.ensure(static_cast<size_t>(E) * 4));
  DCK(S.l_stepping.ensure(static_cast<size_t>(E) * 4 + 16));
  DCK(S.l_around.ensure(static_cast<size_t>(E) * 4));
  DCK(S.l_astate.ensure(static_cast<size_t>(E) * 4));
  DCK(S.l_aW.ensure(static_cast<size_t>(kAsyncK) * E * 4));
  DCK(S.l_aP.ensure(static_cast<size_t>(kAsyncK) * E * 4));
  DCK(S.l_spec.ensure(static_cast<size_t>(E) * 16 + 16));
  if (E >= kWideBackprop) {  // wide-batch backprop: keys / values (x2) + sort scratch, sized before capture
    const int nbp = E * (ctx->params.tree_depth > 0 ? ctx->params.tree_depth : 1);
    size_t scratch = 0;
    DCK(cub::DeviceRadixSort::SortPairs(nullptr, scratch, static_cast<const int*>(nullptr), static_cast<int*>(nullptr),
                                        static_cast<const int*>(nullptr), static_cast<int*>(nullptr), nbp, 0, 32));
    const size_t nn = (static_cast<size_t>(nbp) + 63) / 64 * 64;
    DCK(S.bp_buf.ensure(nn * 4 * 4 + scratch));
  }
  DCK(S.l_actr.ensure(static_cast<size_t>(kAsyncK) * kRingCtr * 4));
  DCK(S.l_adl.ensure(static_cast<size_t>(kAsyncK) * E * 4));
  DCK(S.l_fin.ensure(static_cast<size_t>(E) * 4 + 16));
  DCK(S.l_rsi.ensure(static_cast<size_t>(E) * 4));
  DCK(S.l_ract.ensure(static_cast<size_t>(E) * 4));
  wave_enabled(ctx);  // reads PPG_WAVE / PPG_WAVE_BUDGET / PPG_WAVE_SWITCH
  DCK(ctx->b_counter.ensure(16));  // launch_disc's work counter (no allocation during capture)
  return PPG_SUCCESS;
}

void dt_views(ppg_ctx* ctx, DTreeState& S) {
  DTree& t = S.t;
  t.parent = S.parent.as<int32_t>();
  t.depth = S.depth.as<int32_t>();
  t.q = S.q.as<double>();
  t.visits = S.visits.as<long long>();
  t.vv = S.vv.as<int32_t>();
  t.flags = S.flags.as<uint8_t>();
  t.u_off = S.u_off.as<long long>();
  t.u_n = S.u_n.as<int32_t>();
  t.u_head = S.u_head.as<int32_t>();
  t.c_n = S.c_n.as<int32_t>();
  t.selc = S.selc.as<int32_t>();
  t.action = S.action.as<double>();
  t.poses = S.poses.as<double>();
  t.anc = S.anc.as<int32_t>();
  t.apool = S.apool.as<double>();
  t.cpool = S.cpool.as<int32_t>();
  t.sel_node = S.sel_node.as<int32_t>();
  t.sel_act = S.sel_act.as<long long>();
  t.gp = S.gp.as<double>();
  t.ga = S.ga.as<double>();
  t.cp = S.cp.as<double>();
  t.st = S.st.as<int32_t>();
  t.gr = S.gr.as<uint8_t>();
  t.nu = S.nu.as<int32_t>();
  t.un = S.un.as<double>();
  t.meta = S.meta.as<int32_t>();
  t.rew = S.l_rew.as<unsigned long long>();
  t.logtab = S.logtab.as<double>();
  t.sc = S.sc.as<DTScal>();
  const ppg_params& p = ctx->params;
  t.n_envs = S.n_envs;
  t.n = S.n;
  t.na = S.na;
  t.leaf_parallel = p.leaf_parallel;

  LockArgs& a = S.la;
  a = LockArgs{};
  a.S = ctx->scene;
  a.node_poses = t.cp;
  a.node_meta = t.meta;
  a.n_nodes = S.n_envs;
  a.used = S.n_envs;
  a.used_global = S.n_envs;
  a.env_lo = 0;
  a.leaf_parallel = p.leaf_parallel;
  a.cap = 0;
  a.seed = p.rng_seed;
  a.iteration = 0;
  a.env_node = S.l_node.as<int32_t>();
  a.env_pushes = S.l_pushes.as<int32_t>();
  a.env_done = S.l_done.as<uint8_t>();
  a.env_bygrasp = S.l_byg.as<uint8_t>();
  a.env_harvested = S.l_harv.as<uint8_t>();
  a.env_flag = S.l_flag.as<uint8_t>();
  a.env_reward = S.l_reward.as<double>();
  a.env_poses = S.l_poses.as<double>();
  a.env_push = S.l_push.as<double>();
  a.env_status = S.l_status.as<int32_t>();
  a.n_stepping = S.l_stepping.as<int32_t>();
  a.stepping = S.l_stepping.as<int32_t>() + 4;
  a.mt = S.l_mt.as<uint64_t>();
  a.mt_idx = S.l_mtidx.as<int32_t>();
  a.E = S.n_envs;
  a.W = S.l_W.as<int32_t>();
  a.rew = S.l_rew.as<unsigned long long>();
  a.active = S.l_active.as<int32_t>();
  a.n_active = S.l_nactive.as<int32_t>();
  a.counters = S.l_counters.as<long long>();
  a.dyn = t.sc->lock_dyn;
  a.step_trace = step_trace_buffer(ctx);
  a.env_round = S.l_around.as<int32_t>();
  a.env_state = S.l_astate.as<int32_t>();
  a.a_W = S.l_aW.as<int32_t>();
  a.a_P = S.l_aP.as<int32_t>();
  a.a_spec = speculate_enabled() && S.n_envs <= kSpecMaxEnvs ? S.l_spec.as<int4>() : nullptr;
  a.a_ctr = S.l_actr.as<int32_t>();
  a.a_dl = S.l_adl.as<int32_t>();
  a.a_ctl = t.sc->async_ctl;
  a.a_wcap = S.n_envs;
  a.fin_count = S.l_fin.as<int32_t>();
  a.fin_list = S.l_fin.as<int32_t>() + 4;
  a.resume_si = S.l_rsi.as<int32_t>();
  a.resume_active = S.l_ract.as<uint32_t>();
  a.wave_switch = ctx->wave_switch;
  a.wave_budget = ctx->wave_budget;
  a.round_mode = nullptr;  // set by dt_mode for adaptive graphs
  a.round_guard = &t.sc->round_guard;
  a.hybrid_min = ctx->hybrid_min_envs;
  S.lra = ResolveArgs{ctx->scene, a.env_poses, a.env_push, a.env_poses, a.env_status, nullptr, nullptr, S.n_envs};
  S.lra.idx = a.stepping;
  S.lra.E_dev = a.n_stepping;
  S.C = make_const(ctx->params, S.n, ctx->side, ctx->margin);
}

// One lockstep round (captured into the WHILE body).
// Round mode of the device-tree graph: hybrid-capable batches decide per
// round on the device (the harvest's round_mode flag); every other batch
// has one fixed mode and no flag (so the harvest never writes one).
RoundMode dt_mode(ppg_ctx* ctx, DTreeState& S) {
  RoundMode m = round_mode(ctx, S.n, S.n_envs);
  if (m == RoundMode::kHybrid && ctx->hybrid_min_envs > 0) m = RoundMode::kAdaptive;
  S.la.round_mode = m == RoundMode::kAdaptive ? &S.t.sc->round_mode : nullptr;
  return m;
}

// One WHILE-body round: a lockstep round, or (warp mode / the warp half of
// adaptive mode) the asynchronous lockstep, which runs every remaining round
// of the call (its kernels return at once when the harvest picked hybrid).
int dt_round(ppg_ctx* ctx, DTreeState& S, cudaStream_t st, RoundMode m) {
  if (async_enabled(ctx) && (m == RoundMode::kWarp || m == RoundMode::kAdaptive)) {
    if (m == RoundMode::kAdaptive) {
      // the large-batch half: wave rounds (harvest, sample, budgeted physics,
      // post) or barrier hybrid rounds; their kernels return at once when the
      // call runs asynchronously (round_mode 0)
      const int rc = wave_enabled(ctx) ? launch_wave(ctx, S.C, S.la, S.lra, S.n_envs, st)
                                       : lock_round_on(ctx, S.C, S.la, S.lra, S.n_envs, RoundMode::kHybrid, st);
      if (rc != PPG_SUCCESS) return rc;
    }
    return launch_async(ctx, S.C, S.la, S.n_envs, st, false);
  }
  return lock_round_on(ctx, S.C, S.la, S.lra, S.n_envs, m, st);
}

// select -> gather -> expand -> attach -> recount -> copy: the part of an
// iteration before batch_simulate (launched into a capturing stream).
int dt_launch_pre(ppg_ctx* ctx, DTreeState& S, cudaStream_t st) {
  const int E = S.n_envs, n = S.n;
  // large disc batches expand "hybrid": the pushes on the lane-per-env disc
  // kernel (throughput), the children's untried lists and grasp flags one
  // warp per pair (a lane-per-pair sampler walks its candidates serially)
  const bool hybrid = ctx->scene_all_discs && n <= kDiscMaxN && ctx->disc_kernels && !ctx->warp_max_explicit &&
                      ctx->hybrid_min_envs > 0 && E >= ctx->hybrid_min_envs;
  const bool warp = !hybrid && use_warp(ctx, ctx->scene_all_discs, n, E, true);
  const bool disc = !warp && use_disc(ctx, ctx->scene_all_discs, n);
  const int gg = std::max(1, std::min(4 * ctx->num_sms, (E * n * 3 + 255) / 256));
  const DTree& t = S.t;
  dt_select_kernel<<<1, kSelThreads, 0, st>>>(t);
  dt_gather_kernel<<<gg, 256, 0, st>>>(t, disc);
  {
    ExpandArgs a{ctx->scene, t.gp, t.ga, t.cp, t.st, t.gr, t.nu, t.un, E};
    a.P_dev = &t.sc->n_pairs;
    if (warp) {
      PPG_WARP_LAUNCH(expand_warp_kernel, !ctx->scene_all_discs, n, E, st, S.C, a);
    } else if (disc) {
      ResolveArgs ra{ctx->scene, t.cp, t.ga, t.cp, t.st, nullptr, nullptr, E};
      ra.E_dev = &t.sc->n_pairs;
      const int rc = launch_disc(ctx, S.C, ra, n, E, st);
      if (rc != PPG_SUCCESS) return rc;
      if (hybrid)
        expand_post_warp_kernel<false><<<(E + kWarpsPerBlock - 1) / kWarpsPerBlock, kWarpsPerBlock * 32, 0, st>>>(S.C, a);
      else
        expand_post_kernel<<<(E + kBlock - 1) / kBlock, kBlock, smem_for(n), st>>>(S.C, a);
    } else {
      expand_kernel<<<(E + kBlock - 1) / kBlock, kBlock, smem_for(n), st>>>(S.C, a);
    }
    DCK(cudaGetLastError());
  }
  dt_attach_kernel<<<1, 1024, 0, st>>>(t);
  dt_recount_kernel<<<1, 1024, 0, st>>>(t);
  dt_copy_kernel<<<gg, 256, 0, st>>>(t);
  DCK(cudaGetLastError());
  return PPG_SUCCESS;
}

// backprop of an iteration (pmbs.cpp:236-240): one warp stepping the pairs
// in batch order, or for wide batches the pairs regrouped by ancestor
// (dt_bp_keys_kernel + a stable radix sort + dt_bp_fold_kernel).  Called
// while capturing: the sort's scratch is sized here.
int dt_launch_backprop(ppg_ctx* ctx, DTreeState& S, cudaStream_t st) {
  const int E = S.n_envs;
  const int dmax = ctx->params.tree_depth > 0 ? ctx->params.tree_depth : 1;
  if (E < kWideBackprop) {
    dt_backprop_kernel<<<1, 32, 0, st>>>(S.t);
    DCK(cudaGetLastError());
    return PPG_SUCCESS;
  }
  const int n = E * dmax;
  size_t scratch = 0;  // (the buffer was sized with this query before capture)
  DCK(cub::DeviceRadixSort::SortPairs(nullptr, scratch, static_cast<const int*>(nullptr), static_cast<int*>(nullptr),
                                      static_cast<const int*>(nullptr), static_cast<int*>(nullptr), n, 0, 32, st));
  const size_t nn = (static_cast<size_t>(n) + 63) / 64 * 64;
  if (S.bp_buf.cap < nn * 4 * 4 + scratch) {
    ctx->err = "device tree: backprop scratch not reserved";
    return PPG_EINVAL;
  }
  int* k_in = S.bp_buf.as<int>();
  int* k_out = k_in + nn;
  int* v_in = k_out + nn;
  int* v_out = v_in + nn;
  dt_bp_keys_kernel<<<(n + 255) / 256, 256, 0, st>>>(S.t, dmax, k_in, v_in);
  DCK(cudaGetLastError());
  DCK(cub::DeviceRadixSort::SortPairs(v_out + nn, scratch, k_in, k_out, v_in, v_out, n, 0, 32, st));
  dt_bp_fold_kernel<<<(n + 255) / 256, 256, 0, st>>>(S.t, k_out, v_out, n);
  DCK(cudaGetLastError());
  return PPG_SUCCESS;
}

// With a simulate hook installed (the sharded multi-GPU driver) an iteration
// is two graphs around the host call: pre (above) and post (backprop, stop).
int dt_capture_hooked(ppg_ctx* ctx, DTreeState& S) {
  cudaStream_t st = ctx->stream;
  S.la.cond = 0;
  S.la.round_mode = nullptr;
  DCK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  int rc = dt_launch_pre(ctx, S, st);
  cudaGraph_t g = nullptr;
  const cudaError_t e = cudaStreamEndCapture(st, &g);
  if (rc != PPG_SUCCESS) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  DCK(e);
  S.graph = g;
  DCK(cudaGraphInstantiate(&S.exec, S.graph, 0));
  DCK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  if (const int brc = dt_launch_backprop(ctx, S, st); brc != PPG_SUCCESS) return brc;
  dt_stop_kernel<<<1, 1, 0, st>>>(S.t);
  DCK(cudaStreamEndCapture(st, &S.graph_post));
  DCK(cudaGraphInstantiate(&S.exec_post, S.graph_post, 0));
  return PPG_SUCCESS;
}

// Captures one PMBS iteration as a graph (select -> expand -> attach ->
// lockstep WHILE -> backprop -> stop).
int dt_capture(ppg_ctx* ctx, DTreeState& S) {
  cudaStream_t st = ctx->stream;
  const int E = S.n_envs;
  if (!S.st2) DCK(cudaStreamCreateWithFlags(&S.st2, cudaStreamNonBlocking));
  DCK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  cudaStreamCaptureStatus cs;
  cudaGraph_t g = nullptr;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  DCK(cudaStreamGetCaptureInfo(st, &cs, nullptr, &g, &deps, &nd));
  cudaGraphConditionalHandle cond;
  DCK(cudaGraphConditionalHandleCreate(&cond, g, 0, 0));
  S.la.cond = cond;
  const RoundMode mode = dt_mode(ctx, S);
  const DTree& t = S.t;
  {
    const int rc = dt_launch_pre(ctx, S, st);
    if (rc != PPG_SUCCESS) return rc;
  }
  lock_init_kernel<<<(E + 255) / 256, 256, 0, st>>>(S.C, S.la);
  lock_harvest_kernel<<<1, 1024, 0, st>>>(S.C, S.la);
  DCK(cudaGetLastError());
  // lockstep rounds: WHILE (n_active > 0) { round; harvest }
  DCK(cudaStreamGetCaptureInfo(st, &cs, nullptr, &g, &deps, &nd));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = cond;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t wnode;
  DCK(cudaGraphAddNode(&wnode, g, deps, nd, &cp));
  DCK(cudaStreamUpdateCaptureDependencies(st, &wnode, 1, cudaStreamSetCaptureDependencies));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  DCK(cudaStreamBeginCaptureToGraph(S.st2, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  int rc = dt_round(ctx, S, S.st2, mode);
  lock_harvest_kernel<<<1, 1024, 0, S.st2>>>(S.C, S.la);
  cudaGraph_t body_out = nullptr;
  const cudaError_t e2 = cudaStreamEndCapture(S.st2, &body_out);
  if (rc != PPG_SUCCESS) return rc;
  DCK(e2);
  if (const int brc = dt_launch_backprop(ctx, S, st); brc != PPG_SUCCESS) return brc;
  dt_stop_kernel<<<1, 1, 0, st>>>(t);
  DCK(cudaGetLastError());
  DCK(cudaStreamEndCapture(st, &S.graph));
  DCK(cudaGraphInstantiate(&S.exec, S.graph, 0));
  return PPG_SUCCESS;
}

// Debug path (PPG_DTREE_DEBUG=1): the same iteration launched kernel by
// kernel with a synchronize + error check after each, the lockstep loop
// driven from the host.
int dt_iteration_debug(ppg_ctx* ctx, DTreeState& S) {
  cudaStream_t st = ctx->stream;
  const int E = S.n_envs, n = S.n;
  // large disc batches expand "hybrid": the pushes on the lane-per-env disc
  // kernel (throughput), the children's untried lists and grasp flags one
  // warp per pair (a lane-per-pair sampler walks its candidates serially)
  const bool hybrid = ctx->scene_all_discs && n <= kDiscMaxN && ctx->disc_kernels && !ctx->warp_max_explicit &&
                      ctx->hybrid_min_envs > 0 && E >= ctx->hybrid_min_envs;
  const bool warp = !hybrid && use_warp(ctx, ctx->scene_all_discs, n, E, true);
  const bool disc = !warp && use_disc(ctx, ctx->scene_all_discs, n);
  const int gg = std::max(1, std::min(4 * ctx->num_sms, (E * n * 3 + 255) / 256));
  const DTree& t = S.t;
  S.la.cond = 0;
  const RoundMode mode = dt_mode(ctx, S);
#define DSTEP(name, launch)                                                              \
  do {                                                                                   \
    launch;                                                                              \
    cudaError_t e_ = cudaStreamSynchronize(st);                                          \
    if (e_ == cudaSuccess) e_ = cudaGetLastError();                                      \
    if (e_ != cudaSuccess) {                                                             \
      ctx->err = std::string("dtree debug: ") + name + ": " + cudaGetErrorString(e_);    \
      return PPG_ECUDA;                                                                  \
    }                                                                                    \
  } while (0)
  DSTEP("select", (dt_select_kernel<<<1, kSelThreads, 0, st>>>(t)));
  DSTEP("gather", (dt_gather_kernel<<<gg, 256, 0, st>>>(t, disc)));
  {
    ExpandArgs a{ctx->scene, t.gp, t.ga, t.cp, t.st, t.gr, t.nu, t.un, E};
    a.P_dev = &t.sc->n_pairs;
    if (warp) {
      DSTEP("expand_warp", PPG_WARP_LAUNCH(expand_warp_kernel, !ctx->scene_all_discs, n, E, st, S.C, a));
    } else if (disc) {
      ResolveArgs ra{ctx->scene, t.cp, t.ga, t.cp, t.st, nullptr, nullptr, E};
      ra.E_dev = &t.sc->n_pairs;
      DSTEP("expand_disc", launch_disc(ctx, S.C, ra, n, E, st));
      DSTEP("expand_post", (expand_post_kernel<<<(E + kBlock - 1) / kBlock, kBlock, smem_for(n), st>>>(S.C, a)));
    } else {
      DSTEP("expand", (expand_kernel<<<(E + kBlock - 1) / kBlock, kBlock, smem_for(n), st>>>(S.C, a)));
    }
  }
  DSTEP("attach", (dt_attach_kernel<<<1, 1024, 0, st>>>(t)));
  DSTEP("recount", (dt_recount_kernel<<<1, 1024, 0, st>>>(t)));
  DSTEP("copy", (dt_copy_kernel<<<gg, 256, 0, st>>>(t)));
  DSTEP("lock_init", (lock_init_kernel<<<(E + 255) / 256, 256, 0, st>>>(S.C, S.la)));
  for (;;) {
    DSTEP("harvest", (lock_harvest_kernel<<<1, 1024, 0, st>>>(S.C, S.la)));
    int act = 0;
    DCK(cudaMemcpy(&act, S.la.n_active, 4, cudaMemcpyDeviceToHost));
    if (act == 0) break;
    DSTEP("round", dt_round(ctx, S, st, mode));
  }
  DSTEP("backprop", (dt_launch_backprop(ctx, S, st)));
  DSTEP("stop", (dt_stop_kernel<<<1, 1, 0, st>>>(t)));
#undef DSTEP
  return PPG_SUCCESS;
}

std::string signature(const std::vector<int32_t>& depth, const std::vector<double>& action,
                      const std::vector<long long>& visits, const std::vector<double>& q,
                      const std::vector<uint8_t>& flags, const std::vector<long long>& coff,
                      const std::vector<int32_t>& c_n, const std::vector<int32_t>& kids) {
  // pre-order, children in insertion order (mcts.cpp:284-300): the node
  // order first, then the lines formatted in parallel chunks (the %.17g
  // formatting is the cost: ~28K nodes for a 64K-env C4 decision)
  std::vector<int> order;
  order.reserve(depth.size());
  {
    std::vector<std::pair<int, int>> stack{{0, 0}};
    order.push_back(0);
    while (!stack.empty()) {
      auto& [x, k] = stack.back();
      if (k < c_n[x]) {
        const int ch = kids[coff[x] + k];
        ++k;
        order.push_back(ch);
        stack.push_back({ch, 0});
      } else {
        stack.pop_back();
      }
    }
  }
  const size_t N = order.size();
  auto format = [&](size_t lo, size_t hi, std::string& out) {
    char buf[256];
    out.reserve((hi - lo) * 112);
    for (size_t i = lo; i < hi; ++i) {
      const int x = order[i];
      const int len = std::snprintf(buf, sizeof buf, "%d|%.17g,%.17g,%.17g,%.17g|%ld|%.17g|%c%c\n", depth[x],
                                    action[x * 4], action[x * 4 + 1], action[x * 4 + 2], action[x * 4 + 3],
                                    static_cast<long>(visits[x]), q[x], (flags[x] & 1) ? 'g' : '.',
                                    (flags[x] & 2) ? 'd' : '.');
      out.append(buf, static_cast<size_t>(len));
    }
  };
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const size_t T = std::min<size_t>(std::min<size_t>(hw, 32), N / 1024);
  if (T < 2) {
    std::string out;
    format(0, N, out);
    return out;
  }
  std::vector<std::string> parts(T);
  std::vector<std::thread> th;
  for (size_t t = 0; t < T; ++t) th.emplace_back(format, N * t / T, N * (t + 1) / T, std::ref(parts[t]));
  for (auto& x : th) x.join();
  size_t total = 0;
  for (const auto& p : parts) total += p.size();
  std::string out;
  out.reserve(total);
  for (const auto& p : parts) out += p;
  return out;
}

}  // namespace

namespace {

// Search start (SearchTree::create, mcts.cpp:28-39, + run_pmbs setup,
// pmbs.cpp:242-260): root sample_pushes / graspable, tree + batch buffers,
// the graph key (graphs are re-captured when the configuration changes) and
// the root node + scalars on the device.
int dt_begin(ppg_ctx* ctx, const double* root_poses, bool sharded) {
  const ppg_params& p = ctx->params;
  if (p.n_envs < 1) {
    ctx->err = "n_envs must be >= 1";
    return PPG_EINVAL;
  }
  if (p.tree_depth + 1 >= kMaxTreeDepth || p.tree_depth + p.rollout_depth + 1 >= kMaxGammaPow) {
    ctx->err = "device tree: tree_depth too large";
    return PPG_EINVAL;
  }
  DCK(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  const int n = ctx->scene.n, na = p.pushes_per_object;
  // root: sample_pushes + graspable (SearchTree::create, mcts.cpp:28-39)
  std::vector<double> root_untried(static_cast<size_t>(n) * na * 4);
  int32_t cnt = 0;
  uint8_t rg = 0;
  const double* root_list_dev = nullptr;  // the list left on the device (warp path), else in root_untried
  int rc = ppg_root_sample_grasp(ctx, root_poses, root_untried.data(), &cnt, &rg, &root_list_dev);
  if (rc != PPG_SUCCESS) return rc;
  if (cnt == 0) {
    ctx->err = "no legal push action at the root";
    return PPG_ENOLEGAL;
  }
  if (!ctx->dtree) ctx->dtree = new DTreeState;
  DTreeState& S = *ctx->dtree;
  S.last_valid = false;
  {
    // everything baked into the captured graph: parameters (minus the
    // per-search values kept in DTScal), scene tables
    ppg_params kp = p;
    kp.rng_seed = 0;
    kp.c_explore = 0.0;
    kp.budget_iterations = 0;
    kp.max_iterations = 0;
    kp.max_seconds = 0.0;
    std::string key(reinterpret_cast<const char*>(&kp), sizeof kp);
    key.append(reinterpret_cast<const char*>(&ctx->scene), sizeof ctx->scene);
    key.append(reinterpret_cast<const char*>(&ctx->side), sizeof ctx->side);
    key.append(reinterpret_cast<const char*>(&ctx->margin), sizeof ctx->margin);
    // kernel-mode inputs (which kernels the graph holds)
    const int modes[8] = {ctx->scene_all_discs ? 1 : 0, ctx->force_generic ? 1 : 0, ctx->warp_poly ? 1 : 0,
                          ctx->warp_max_envs, ctx->warp_max_explicit ? 1 : 0, ctx->disc_kernels ? 1 : 0,
                          ctx->hybrid_min_envs, (ctx->sim_hook ? 1 : 0) | (sharded ? 2 : 0)};
    key.append(reinterpret_cast<const char*>(modes), sizeof modes);
    if (S.key != key) S.release_graph();
    S.key = key;
  }
  if (S.n != n) {  // per-node pose rows change size: start the tree buffers afresh
    DevBuf* node_bufs[] = {&S.parent, &S.depth, &S.q, &S.visits, &S.vv, &S.flags, &S.u_off, &S.u_n, &S.u_head,
                           &S.c_n, &S.selc, &S.action, &S.poses, &S.anc, &S.apool, &S.cpool};
    DCK(cudaStreamSynchronize(st));
    for (DevBuf* b : node_bufs) b->release();
    S.cap_nodes = 0;
    S.cap_actions = 0;
    S.release_graph();
  }
  S.n_envs = p.n_envs;
  S.n = n;
  S.na = na;
  if (S.logtab.cap < (static_cast<size_t>(S.cap_nodes) + p.n_envs + 2) * 8) {  // log table covers visits + n_envs
    S.cap_nodes = 0;  // forces dt_reserve to re-grow (contents preserved up to used = 0: fresh search)
  }
  {
    int want = 1 + p.n_envs * (p.budget_iterations ? std::min<long long>(p.max_iterations, 64) : 8);
    if (const char* cn = std::getenv("PPG_DTREE_NODES")) want = std::max(want, std::atoi(cn));
    want = std::max(want, 1 + 2 * p.n_envs);
    if ((rc = dt_reserve(ctx, S, 0, 0, want, static_cast<long long>(want) * n * na)) != PPG_SUCCESS) return rc;
  }
  if ((rc = dt_batch(ctx, S)) != PPG_SUCCESS) return rc;
  dt_views(ctx, S);
  // root node + scalars: one staged block, one copy, one kernel
  {
    DTScal h;
    std::memset(&h, 0, sizeof h);
    h.n_nodes = 1;
    h.dT = p.tree_depth;
    h.dS = p.rollout_depth;
    h.es_level = 1;
    h.min_grasp_depth = INT_MAX;
    h.levels = 1;
    h.stop = -1;
    h.a_used = cnt;
    h.unsettled[0] = rg ? 0 : 1;  // root: non-terminal with untried actions unless graspable
    h.max_iters = p.budget_iterations ? static_cast<int>(p.max_iterations) : 0;
    h.c_explore = p.c_explore;
    h.lock_dyn[4] = static_cast<int>(static_cast<uint32_t>(p.rng_seed));
    h.lock_dyn[5] = static_cast<int>(static_cast<uint32_t>(p.rng_seed >> 32));
    const size_t bytes = sizeof(DTScal) + 8 + static_cast<size_t>(n) * 24;
    char* hp = S.pinned(bytes);
    if (!hp) {
      ctx->err = "device tree: pinned staging allocation failed";
      return PPG_ECUDA;
    }
    DCK(cudaStreamSynchronize(st));  // the previous search's reads of the staging block are done
    std::memcpy(hp, &h, sizeof h);
    const int rf = rg ? 1 : 0;  // dead needs untried.empty(): cnt > 0 here
    std::memcpy(hp + sizeof h, &rf, 4);
    std::memcpy(hp + sizeof h + 8, root_poses, static_cast<size_t>(n) * 24);
    DCK(S.dstage.ensure(bytes));
    DCK(cudaMemcpyAsync(S.dstage.p, hp, bytes, cudaMemcpyHostToDevice, st));
    dt_root_kernel<<<1, 128, 0, st>>>(S.t, S.dstage.as<char>(), n, cnt, S.la.counters);
    DCK(cudaGetLastError());
    if (root_list_dev) {
      DCK(cudaMemcpyAsync(S.t.apool, root_list_dev, static_cast<size_t>(cnt) * 32, cudaMemcpyDeviceToDevice, st));
    } else {
      DCK(cudaMemcpyAsync(S.t.apool, root_untried.data(), static_cast<size_t>(cnt) * 32, cudaMemcpyHostToDevice,
                          st));
    }
  }
  return PPG_SUCCESS;
}

// Reads the final tree back once: best_root_child (mcts.cpp:218-235), the
// tree signature (mcts.cpp:284-300) and the statistics.  ctr = rollout steps,
// rounds, re-purposes, resolve calls of the whole search.
int dt_finish(ppg_ctx* ctx, const DTScal& h, int stop, double elapsed_s, double loop_s, const int64_t* ctr_in,
              double* action_out, ppg_search_stats* stats, char* sig_buf, int64_t sig_cap, int64_t* sig_len) {
  DTreeState& S = *ctx->dtree;
  const ppg_params& p = ctx->params;
  cudaStream_t st = ctx->stream;
  int64_t ctr[4] = {ctr_in[0], ctr_in[1], ctr_in[2], ctr_in[3]};
  if (S.la.step_trace) step_trace_dump(ctx);
  S.last_valid = false;
  if (stop == 3) {
    ctx->err = "device tree: selection invariant violated";
    return PPG_EINVAL;
  }
  S.last_valid = true;
  S.last_nodes = h.n_nodes;
  S.last_a_used = h.a_used;
  S.last_dT = h.dT;
  S.last_dS = h.dS;
  S.last_es = h.es_level;
  // read the tree back once
  const int N = h.n_nodes;
  std::vector<int32_t> depth(N), c_n(N), kids(static_cast<size_t>(N > 1 ? N - 1 : 1));
  std::vector<double> q(N), action(static_cast<size_t>(N) * 4);
  std::vector<long long> visits(N), coff(N);
  std::vector<uint8_t> flags(N);
  {  // one pinned staging block: every copy asynchronous, one synchronisation.
     // Large trees: the children lists gathered densely on the device (the
     // children pool is action-sized); small trees: the pool itself.
    const bool dense = h.a_used > (1 << 18);
    const size_t Nn = (static_cast<size_t>(N) + 63) / 64 * 64;
    int* d_kids = nullptr;
    if (dense) {
      size_t scan_bytes = 0;
      DCK(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, static_cast<const int*>(nullptr),
                                        static_cast<int*>(nullptr), N, st));
      DCK(S.dstage.ensure(Nn * 4 * 2 + scan_bytes));
      int* d_coff = S.dstage.as<int>();
      d_kids = d_coff + Nn;
      DCK(cub::DeviceScan::ExclusiveSum(d_kids + Nn, scan_bytes, S.t.c_n, d_coff, N, st));
      dt_kids_kernel<<<std::min(1024, (N + 255) / 256), 256, 0, st>>>(S.t, N, d_coff, d_kids);
      DCK(cudaGetLastError());
    }
    std::vector<long long> u_off(dense ? 0 : N);
    std::vector<int32_t> cpool(dense ? 0 : static_cast<size_t>(h.a_used));
    const size_t nk = N > 1 ? static_cast<size_t>(N - 1) : 0;
    const size_t seg[8] = {N * 4ull, N * 4ull, N * 8ull, N * 32ull, N * 8ull, static_cast<size_t>(N),
                           dense ? nk * 4 : static_cast<size_t>(h.a_used) * 4, dense ? 0 : N * 8ull};
    const void* dsrc[8] = {S.t.depth, S.t.c_n, S.t.q, S.t.action, S.t.visits, S.t.flags,
                           dense ? static_cast<const void*>(d_kids) : static_cast<const void*>(S.t.cpool), S.t.u_off};
    void* hdst[8] = {depth.data(), c_n.data(), q.data(), action.data(), visits.data(), flags.data(),
                     dense ? static_cast<void*>(kids.data()) : static_cast<void*>(cpool.data()), u_off.data()};
    size_t off[8], total = 0;
    for (int i = 0; i < 8; ++i) {
      off[i] = total;
      total += (seg[i] + 15) / 16 * 16;
    }
    DCK(cudaStreamSynchronize(st));  // earlier users of the staging block are done
    char* hp = S.pinned(total);
    if (!hp) {
      ctx->err = "device tree: pinned staging allocation failed";
      return PPG_ECUDA;
    }
    for (int i = 0; i < 8; ++i)
      if (seg[i]) DCK(cudaMemcpyAsync(hp + off[i], dsrc[i], seg[i], cudaMemcpyDeviceToHost, st));
    DCK(cudaStreamSynchronize(st));
    for (int i = 0; i < 8; ++i)
      if (seg[i]) std::memcpy(hdst[i], hp + off[i], seg[i]);
    long long acc = 0;
    for (int x = 0; x < N; ++x) {
      coff[x] = acc;
      if (!dense)
        for (int k = 0; k < c_n[x]; ++k) kids[acc + k] = cpool[u_off[x] + k];
      acc += c_n[x];
    }
  }
  // best_root_child (mcts.cpp:218-235)
  int best = -1;
  double best_score = -std::numeric_limits<double>::infinity();
  long long best_visits = -1;
  for (int k = 0; k < c_n[0]; ++k) {
    const int ch = kids[coff[0] + k];
    if (visits[ch] == 0) continue;
    const double score = p.rank_by_ucb ? ucb_score_host(q[ch], static_cast<long>(visits[ch]), static_cast<long>(visits[0]),
                                                        p.c_explore)
                                       : q[ch] / static_cast<double>(visits[ch]);
    if (score > best_score || (score == best_score && visits[ch] > best_visits)) {
      best_score = score;
      best_visits = visits[ch];
      best = ch;
    }
  }
  if (best < 0) {
    ctx->err = "search produced no evaluated root child";
    return PPG_EINVAL;
  }
  std::memcpy(action_out, &action[static_cast<size_t>(best) * 4], 32);
  const std::string sig = signature(depth, action, visits, q, flags, coff, c_n, kids);
  if (stats) {
    ppg_search_stats s;
    std::memset(&s, 0, sizeof s);
    s.iterations = h.iteration;
    s.expansions = h.expansions;
    s.elapsed_s = elapsed_s;
    s.stop_reason = stop;
    s.final_tree_depth = h.dT;
    s.env_steps = ctr[3] + h.expansions;
    s.rollout_steps = ctr[0];
    s.lockstep_rounds = ctr[1];
    s.signature_fnv = fnv1a(sig);
    s.n_nodes = N;
    s.simulate_s = loop_s;  // one graph per iteration: the phases are not timed separately
    *stats = s;
  }
  if (sig_len) *sig_len = static_cast<int64_t>(sig.size());
  if (sig_buf && sig_cap > 0) {
    const size_t m = sig.size() < static_cast<size_t>(sig_cap - 1) ? sig.size() : static_cast<size_t>(sig_cap - 1);
    std::memcpy(sig_buf, sig.data(), m);
    sig_buf[m] = '\0';
  }
  return PPG_SUCCESS;
}

// Sharded iteration graphs (multi-GPU, multi.cu): pre = select -> expand ->
// attach -> copy -> lock_init -> local harvest half; round = one lockstep
// round over this shard's active envs -> local harvest half; post = backprop
// -> stop.  Between them the host enqueues the per-round W exchange and the
// apply half of the harvest (lock_harvest_apply_kernel), which writes `go`.
int dt_capture_sharded(ppg_ctx* ctx, DTreeState& S, int work) {
  cudaStream_t st = ctx->stream;
  const int E = S.n_envs;
  S.la.cond = 0;
  const RoundMode mode = dt_mode(ctx, S);
  DCK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  int rc = dt_launch_pre(ctx, S, st);
  if (rc == PPG_SUCCESS) {
    lock_init_kernel<<<(E + 255) / 256, 256, 0, st>>>(S.C, S.la);
    lock_harvest_local_kernel<<<1, 1024, 0, st>>>(S.C, S.la);
  }
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture(st, &g);
  if (rc != PPG_SUCCESS) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  DCK(e);
  S.graph = g;
  DCK(cudaGraphInstantiate(&S.exec, S.graph, 0));
  DCK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  rc = lock_round_on(ctx, S.C, S.la, S.lra, work, mode, st);
  if (rc == PPG_SUCCESS) lock_harvest_local_kernel<<<1, 1024, 0, st>>>(S.C, S.la);
  g = nullptr;
  e = cudaStreamEndCapture(st, &g);
  if (rc != PPG_SUCCESS) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  DCK(e);
  S.graph_round = g;
  DCK(cudaGraphInstantiate(&S.exec_round, S.graph_round, 0));
  DCK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  if (const int brc = dt_launch_backprop(ctx, S, st); brc != PPG_SUCCESS) return brc;
  dt_stop_kernel<<<1, 1, 0, st>>>(S.t);
  DCK(cudaStreamEndCapture(st, &S.graph_post));
  DCK(cudaGraphInstantiate(&S.exec_post, S.graph_post, 0));
  return PPG_SUCCESS;
}

}  // namespace

// run_pmbs (pmbs.cpp:242-292) with the rollout batch sharded over the
// context's group (multi.cu).  Every shard holds an identical device tree
// (select / expand / attach / backprop replicated on identical data); each
// iteration's lockstep is split by environment with ONE W exchange per round
// and one reward max at the end, so the decision and the tree are
// bit-identical to the single-GPU search for any shard count.
namespace ppg {

int run_pmbs_sharded(ppg_ctx* ctx, const double* root_poses, double* action_out, ppg_search_stats* stats,
                     char* sig_buf, int64_t sig_cap, int64_t* sig_len) {
  Group* g = ctx->group;
  const int M = group_size(g), G = group_world(g), r0 = group_rank0(g);
  const auto t_start = std::chrono::steady_clock::now();
  const auto elapsed = [&t_start] {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
  };
  const ppg_params& p = ctx->params;
  const int work = (p.n_envs + G - 1) / G;  // the largest shard
  std::vector<ppg_ctx*> m(M);
  for (int k = 0; k < M; ++k) m[k] = group_member(g, k);
  const auto set_shard = [&](int k) {
    DTreeState& S = *m[k]->dtree;
    S.la.shard_r = r0 + k;
    S.la.shard_g = G;
    S.la.go = m[k]->l_go.as<int32_t>();
    // the apply kernel runs outside the graphs: it must carry the adaptive
    // round-mode flag the captured round graph reads (dt_views cleared it)
    dt_mode(m[k], S);
  };
  for (int k = 0; k < M; ++k) {
    ppg_ctx* c = m[k];
    int rc = dt_begin(c, root_poses, true);
    if (rc != PPG_SUCCESS) {
      ctx->err = c->err;
      return rc;
    }
    if (c->l_go.ensure(16) != cudaSuccess || (!c->h_go && cudaMallocHost(&c->h_go, 16) != cudaSuccess)) {
      ctx->err = "sharded run_pmbs: allocation failed";
      return PPG_ECUDA;
    }
    set_shard(k);
  }
  bool waves = true;
  for (int k = 0; k < M; ++k) waves = waves && shard_waves_enabled(m[k]);
  std::vector<DTScal> h(M);
  std::vector<int32_t*> wb(M);
  std::vector<unsigned long long*> rb(M), vb(M);
  std::vector<long long*> cb(M);
  int stop = -1;
  const long long per_iter_actions = static_cast<long long>(p.n_envs) * m[0]->dtree->n * m[0]->dtree->na;
  const auto t_loop = std::chrono::steady_clock::now();
  int rc = PPG_SUCCESS;
  for (;;) {
    for (int k = 0; k < M; ++k) {
      DTreeState& S = *m[k]->dtree;
      DCK(cudaSetDevice(m[k]->device));
      DCK(cudaMemcpyAsync(&h[k], S.t.sc, sizeof(DTScal), cudaMemcpyDeviceToHost, m[k]->stream));
      DCK(cudaStreamSynchronize(m[k]->stream));
      if (h[k].round_guard < 0 || h[k].err[0]) {
        ctx->err = "sharded device tree: lockstep round limit or corrupt ancestor row";
        return PPG_EINVAL;
      }
      if (h[k].stop != h[0].stop || h[k].iteration != h[0].iteration || h[k].n_nodes != h[0].n_nodes) {
        ctx->err = "sharded device tree: shards diverged";
        return PPG_EINVAL;
      }
    }
    if (h[0].stop >= 0) {
      stop = h[0].stop;
      break;
    }
    if (!p.budget_iterations && h[0].iteration > 0) {
      // seconds budget: every shard must stop at the same iteration, so the
      // shards vote (max) instead of each reading its own clock
      const unsigned long long vote = elapsed() >= p.max_seconds ? 1ull : 0ull;
      for (int k = 0; k < M; ++k) {
        vb[k] = reinterpret_cast<unsigned long long*>(m[k]->l_go.as<char>() + 8);
        DCK(cudaSetDevice(m[k]->device));
        DCK(cudaMemcpyAsync(vb[k], &vote, 8, cudaMemcpyHostToDevice, m[k]->stream));
      }
      if ((rc = group_allreduce_max_u64(ctx, g, vb.data(), 1)) != PPG_SUCCESS) return rc;
      for (int k = 0; k < M; ++k) {
        DCK(cudaSetDevice(m[k]->device));
        DCK(cudaMemcpyAsync(m[k]->h_go + 2, vb[k], 8, cudaMemcpyDeviceToHost, m[k]->stream));
      }
      if ((rc = group_wait(ctx, g)) != PPG_SUCCESS) return rc;
      if (*reinterpret_cast<unsigned long long*>(m[0]->h_go + 2)) {
        stop = 0;
        break;
      }
    }
    for (int k = 0; k < M; ++k) {
      ppg_ctx* c = m[k];
      DTreeState& S = *c->dtree;
      DCK(cudaSetDevice(c->device));
      if (h[k].n_nodes + p.n_envs > S.cap_nodes || h[k].a_used + per_iter_actions > S.cap_actions) {
        const int want = std::max(2 * S.cap_nodes, h[k].n_nodes + p.n_envs);
        const long long wa = std::max(2 * S.cap_actions, h[k].a_used + per_iter_actions);
        if ((rc = dt_reserve(c, S, h[k].n_nodes, h[k].a_used, want, wa)) != PPG_SUCCESS) {
          ctx->err = c->err;
          return rc;
        }
        dt_views(c, S);
        set_shard(k);
      }
      if (!S.exec && (rc = dt_capture_sharded(c, S, work)) != PPG_SUCCESS) {
        cudaStreamCaptureStatus cs;
        if (cudaStreamIsCapturing(c->stream, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) {
          cudaGraph_t junk = nullptr;
          cudaStreamEndCapture(c->stream, &junk);
          if (junk) cudaGraphDestroy(junk);
        }
        cudaGetLastError();
        S.release_graph();
        ctx->err = c->err;
        return rc;
      }
      wb[k] = S.la.W;
      rb[k] = S.la.rew;
      cb[k] = S.la.counters;
      DCK(cudaGraphLaunch(S.exec, c->stream));  // select ... lock_init, local harvest half
      DCK(cudaMemcpyAsync(c->h_go + 2, &S.t.sc->n_pairs, 4, cudaMemcpyDeviceToHost, c->stream));
    }
    if ((rc = group_wait(ctx, g)) != PPG_SUCCESS) return rc;
    const int P = m[0]->h_go[2];
    if (P > 0) {
      for (;;) {
        if ((rc = group_allreduce_sum_i32(ctx, g, wb.data(), static_cast<size_t>(P))) != PPG_SUCCESS) return rc;
        for (int k = 0; k < M; ++k) {
          DTreeState& S = *m[k]->dtree;
          DCK(cudaSetDevice(m[k]->device));
          lock_harvest_apply_kernel<<<1, 1024, 0, m[k]->stream>>>(S.C, S.la);
          DCK(cudaGetLastError());
          DCK(cudaMemcpyAsync(m[k]->h_go, S.la.go, 4, cudaMemcpyDeviceToHost, m[k]->stream));
        }
        if ((rc = group_wait(ctx, g)) != PPG_SUCCESS) return rc;
        const int go = m[0]->h_go[0];
        for (int k = 1; k < M; ++k)
          if (m[k]->h_go[0] != go) {
            ctx->err = "sharded lockstep: shards disagree on termination";
            return PPG_EINVAL;
          }
        if (!go) break;
        if (waves) {  // every remaining round as waves, one exchange per wave (multi.cu)
          std::vector<ShardWave> sw(M);
          for (int k = 0; k < M; ++k) {
            DTreeState& S = *m[k]->dtree;
            sw[k] = ShardWave{m[k], &S.C, S.la, S.lra};
          }
          if ((rc = sharded_wave_rounds(ctx, g, sw, P, work)) != PPG_SUCCESS) return rc;
          break;
        }
        for (int k = 0; k < M; ++k) {
          DCK(cudaSetDevice(m[k]->device));
          DCK(cudaGraphLaunch(m[k]->dtree->exec_round, m[k]->stream));
        }
      }
      if ((rc = group_allreduce_max_u64(ctx, g, rb.data(), static_cast<size_t>(P))) != PPG_SUCCESS) return rc;
    }
    for (int k = 0; k < M; ++k) {
      DCK(cudaSetDevice(m[k]->device));
      DCK(cudaGraphLaunch(m[k]->dtree->exec_post, m[k]->stream));
    }
  }
  const double loop_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_loop).count();
  for (int k = 0; k < M; ++k) cb[k] = m[k]->dtree->la.counters;
  if ((rc = group_allreduce_sum_i64(ctx, g, cb.data(), 4)) != PPG_SUCCESS) return rc;
  int64_t ctr[4];
  DCK(cudaSetDevice(m[0]->device));
  DCK(cudaMemcpyAsync(ctr, cb[0], 32, cudaMemcpyDeviceToHost, m[0]->stream));
  if ((rc = group_wait(ctx, g)) != PPG_SUCCESS) return rc;
  ctr[1] /= G;  // every shard counts every round
  rc = dt_finish(m[0], h[0], stop, elapsed(), loop_s, ctr, action_out, stats, sig_buf, sig_cap, sig_len);
  if (rc != PPG_SUCCESS && m[0] != ctx) ctx->err = m[0]->err;
  return rc;
}

}  // namespace ppg

extern "C" {

// The tree of the last search (SearchResult::tree, mcts.hpp:87-91): see the
// header.  One read of the device tree's node arrays.
int ppg_tree_export(ppg_ctx* ctx, int64_t* n_nodes, int64_t* n_untried, int32_t* parent, int32_t* depth,
                    double* action, int64_t* visits, double* q_sum, uint8_t* flags, double* poses,
                    int32_t* untried_count, double* untried, int32_t* scal) {
  if (!ctx || !n_nodes || !n_untried) return PPG_EINVAL;
  if (!ctx->dtree || !ctx->dtree->last_valid) {
    ctx->err = "tree export: no finished device-tree search on this context";
    return PPG_EINVAL;
  }
  DTreeState& S = *ctx->dtree;
  DCK(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  const int N = S.last_nodes, n = S.n;
  std::vector<long long> u_off(N);
  std::vector<int32_t> u_n(N), u_head(N);
  DCK(cudaMemcpyAsync(u_off.data(), S.u_off.p, N * 8ull, cudaMemcpyDeviceToHost, st));
  DCK(cudaMemcpyAsync(u_n.data(), S.u_n.p, N * 4ull, cudaMemcpyDeviceToHost, st));
  DCK(cudaMemcpyAsync(u_head.data(), S.u_head.p, N * 4ull, cudaMemcpyDeviceToHost, st));
  DCK(cudaStreamSynchronize(st));
  long long U = 0;
  for (int x = 0; x < N; ++x) U += u_n[x] - u_head[x];
  *n_nodes = N;
  *n_untried = U;
  if (parent) DCK(cudaMemcpyAsync(parent, S.parent.p, N * 4ull, cudaMemcpyDeviceToHost, st));
  if (depth) DCK(cudaMemcpyAsync(depth, S.depth.p, N * 4ull, cudaMemcpyDeviceToHost, st));
  if (action) DCK(cudaMemcpyAsync(action, S.action.p, N * 32ull, cudaMemcpyDeviceToHost, st));
  if (visits) DCK(cudaMemcpyAsync(visits, S.visits.p, N * 8ull, cudaMemcpyDeviceToHost, st));
  if (q_sum) DCK(cudaMemcpyAsync(q_sum, S.q.p, N * 8ull, cudaMemcpyDeviceToHost, st));
  if (flags) DCK(cudaMemcpyAsync(flags, S.flags.p, N, cudaMemcpyDeviceToHost, st));
  if (poses) DCK(cudaMemcpyAsync(poses, S.poses.p, static_cast<size_t>(N) * n * 24, cudaMemcpyDeviceToHost, st));
  if (untried_count)
    for (int x = 0; x < N; ++x) untried_count[x] = u_n[x] - u_head[x];
  if (untried) {
    long long k = 0;
    for (int x = 0; x < N; ++x) {
      const int m = u_n[x] - u_head[x];
      if (m > 0)
        DCK(cudaMemcpyAsync(untried + k * 4, S.apool.as<double>() + (u_off[x] + u_head[x]) * 4, m * 32ull,
                            cudaMemcpyDeviceToHost, st));
      k += m;
    }
  }
  DCK(cudaStreamSynchronize(st));
  if (scal) {
    scal[0] = S.last_dT;
    scal[1] = S.last_dS;
    scal[2] = S.last_es;
    scal[3] = n;
  }
  return PPG_SUCCESS;
}

// Test entry (acceptance criterion 3, acceptance.cpp:255-281): loads one
// explicit tree into a scratch device tree and runs the device select_batch
// (dt_select_kernel, the kernel of every PMBS iteration graph) on it.
// Nodes in pre-order with children in insertion order; node x has
// n_children[x] children and n_untried[x] untried actions (none popped).
// Outputs: the selected (node, untried index) pairs in draw order, every
// node's virtual visits after the batch (vv_out), and the sum of virtual
// visits after reset_virtual (pmbs.cpp:65-68; the iteration graph's
// dt_gather_kernel zeroing pass).  *n_sel = 0 is TreeExhausted.
int ppg_debug_select_batch(ppg_ctx* ctx, int n_nodes, const int32_t* parent, const int32_t* depth,
                           const int64_t* visits, const double* q_sum, const uint8_t* flags,
                           const int32_t* n_children, const int32_t* n_untried, int tree_depth, int n_envs,
                           double c_explore, int32_t* sel_node, int32_t* sel_untried, int32_t* n_sel,
                           int64_t* vv_out, int64_t* vsum_after_reset) {
  if (!ctx || n_nodes < 1 || n_envs < 1 || !parent || !depth || !visits || !q_sum || !flags || !n_children ||
      !n_untried || !sel_node || !sel_untried || !n_sel || tree_depth < 0 || tree_depth >= kMaxTreeDepth)
    return PPG_EINVAL;
  DCK(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  const int N = n_nodes;
  // host layout: children (insertion order) then untried entries share u_off
  std::vector<long long> u_off(N), vis(visits, visits + N);
  std::vector<int32_t> u_n(N), u_head(N), c_n(N), cpool, zero(N, 0);
  long long off = 0;
  int max_depth = 0;
  long long max_vis = 0;
  std::vector<int> unsettled(kMaxTreeDepth, 0);
  for (int x = 0; x < N; ++x) {
    if (depth[x] < 0 || depth[x] >= kMaxTreeDepth || (x > 0 && (parent[x] < 0 || parent[x] >= x))) return PPG_EINVAL;
    u_off[x] = off;
    off += n_children[x] + n_untried[x];
    u_n[x] = n_children[x] + n_untried[x];
    u_head[x] = n_children[x];
    c_n[x] = n_children[x];
    max_depth = std::max(max_depth, depth[x]);
    max_vis = std::max(max_vis, static_cast<long long>(visits[x]));
    if (flags[x] == 0 && n_untried[x] > 0) unsettled[depth[x]] += 1;
  }
  cpool.assign(static_cast<size_t>(off > 0 ? off : 1), -1);
  {
    std::vector<int32_t> fill(N, 0);
    for (int x = 1; x < N; ++x) {
      const int p = parent[x];
      if (fill[p] >= n_children[p]) return PPG_EINVAL;
      cpool[u_off[p] + fill[p]++] = x;
    }
    for (int x = 0; x < N; ++x)
      if (fill[x] != n_children[x]) return PPG_EINVAL;
  }
  DevBuf b_parent, b_depth, b_q, b_vis, b_vv, b_flags, b_uoff, b_un, b_uhead, b_cn, b_selc, b_cpool, b_log, b_sc,
      b_seln, b_sela;
  struct Free {
    std::vector<DevBuf*> v;
    ~Free() {
      for (DevBuf* b : v) b->release();
    }
  } fr{{&b_parent, &b_depth, &b_q, &b_vis, &b_vv, &b_flags, &b_uoff, &b_un, &b_uhead, &b_cn, &b_selc, &b_cpool, &b_log,
        &b_sc, &b_seln, &b_sela}};
  DCK(b_parent.ensure(N * 4ull));
  DCK(b_depth.ensure(N * 4ull));
  DCK(b_q.ensure(N * 8ull));
  DCK(b_vis.ensure(N * 8ull));
  DCK(b_vv.ensure(N * 4ull));
  DCK(b_flags.ensure(N));
  DCK(b_uoff.ensure(N * 8ull));
  DCK(b_un.ensure(N * 4ull));
  DCK(b_uhead.ensure(N * 4ull));
  DCK(b_cn.ensure(N * 4ull));
  DCK(b_selc.ensure(N * 4ull));
  DCK(b_cpool.ensure(cpool.size() * 4));
  const size_t lt = static_cast<size_t>(max_vis) + n_envs + 2;
  std::vector<double> tab(lt);
  for (size_t k = 0; k < lt; ++k) tab[k] = std::log(static_cast<double>(k));  // the reference's glibc log
  DCK(b_log.ensure(lt * 8));
  DCK(b_sc.ensure(sizeof(DTScal)));
  DCK(b_seln.ensure(static_cast<size_t>(n_envs) * 4));
  DCK(b_sela.ensure(static_cast<size_t>(n_envs) * 8));
  DCK(cudaMemcpyAsync(b_parent.p, parent, N * 4ull, cudaMemcpyHostToDevice, st));
  DCK(cudaMemcpyAsync(b_depth.p, depth, N * 4ull, cudaMemcpyHostToDevice, st));
  DCK(cudaMemcpyAsync(b_q.p, q_sum, N * 8ull, cudaMemcpyHostToDevice, st));
  DCK(cudaMemcpyAsync(b_vis.p, vis.data(), N * 8ull, cudaMemcpyHostToDevice, st));
  DCK(cudaMemcpyAsync(b_vv.p, zero.data(), N * 4ull, cudaMemcpyHostToDevice, st));
  DCK(cudaMemcpyAsync(b_flags.p, flags, N, cudaMemcpyHostToDevice, st));
  DCK(cudaMemcpyAsync(b_uoff.p, u_off.data(), N * 8ull, cudaMemcpyHostToDevice, st));
  DCK(cudaMemcpyAsync(b_un.p, u_n.data(), N * 4ull, cudaMemcpyHostToDevice, st));
  DCK(cudaMemcpyAsync(b_uhead.p, u_head.data(), N * 4ull, cudaMemcpyHostToDevice, st));
  DCK(cudaMemcpyAsync(b_cn.p, c_n.data(), N * 4ull, cudaMemcpyHostToDevice, st));
  DCK(cudaMemcpyAsync(b_selc.p, zero.data(), N * 4ull, cudaMemcpyHostToDevice, st));
  DCK(cudaMemcpyAsync(b_cpool.p, cpool.data(), cpool.size() * 4, cudaMemcpyHostToDevice, st));
  DCK(cudaMemcpyAsync(b_log.p, tab.data(), lt * 8, cudaMemcpyHostToDevice, st));
  DTScal h;
  std::memset(&h, 0, sizeof h);
  h.n_nodes = N;
  h.dT = tree_depth;
  h.levels = max_depth + 1;
  h.stop = -1;
  h.recompute = 1;  // dt_recount_kernel builds the selectable-children counts
  h.c_explore = c_explore;
  h.min_grasp_depth = INT_MAX;
  for (int d = 0; d < kMaxTreeDepth; ++d) h.unsettled[d] = unsettled[d];
  DCK(cudaMemcpyAsync(b_sc.p, &h, sizeof h, cudaMemcpyHostToDevice, st));
  DTree t{};
  t.parent = b_parent.as<int32_t>();
  t.depth = b_depth.as<int32_t>();
  t.q = b_q.as<double>();
  t.visits = b_vis.as<long long>();
  t.vv = b_vv.as<int32_t>();
  t.flags = b_flags.as<uint8_t>();
  t.u_off = b_uoff.as<long long>();
  t.u_n = b_un.as<int32_t>();
  t.u_head = b_uhead.as<int32_t>();
  t.c_n = b_cn.as<int32_t>();
  t.selc = b_selc.as<int32_t>();
  t.cpool = b_cpool.as<int32_t>();
  t.sel_node = b_seln.as<int32_t>();
  t.sel_act = b_sela.as<long long>();
  t.logtab = b_log.as<double>();
  t.sc = b_sc.as<DTScal>();
  t.n_envs = n_envs;
  dt_recount_kernel<<<1, 1024, 0, st>>>(t);
  dt_select_kernel<<<1, kSelThreads, 0, st>>>(t);
  DCK(cudaGetLastError());
  DCK(cudaMemcpyAsync(&h, b_sc.p, sizeof h, cudaMemcpyDeviceToHost, st));
  std::vector<int32_t> vv(N), sn(n_envs);
  std::vector<long long> sa(n_envs);
  DCK(cudaMemcpyAsync(vv.data(), b_vv.p, N * 4ull, cudaMemcpyDeviceToHost, st));
  DCK(cudaMemcpyAsync(sn.data(), b_seln.p, n_envs * 4ull, cudaMemcpyDeviceToHost, st));
  DCK(cudaMemcpyAsync(sa.data(), b_sela.p, n_envs * 8ull, cudaMemcpyDeviceToHost, st));
  DCK(cudaStreamSynchronize(st));
  if (h.stop == 3) {
    ctx->err = "device select: selection invariant violated";
    return PPG_EINVAL;
  }
  const int P = h.n_pairs;
  *n_sel = P;
  for (int k = 0; k < P; ++k) {
    sel_node[k] = sn[k];
    sel_untried[k] = static_cast<int32_t>(sa[k] - u_off[sn[k]] - n_children[sn[k]]);
  }
  if (vv_out)
    for (int x = 0; x < N; ++x) vv_out[x] = vv[x];
  // reset_virtual: the iteration graph's dt_gather_kernel pass over the nodes
  t.sc = b_sc.as<DTScal>();
  h.n_pairs = 0;
  DCK(cudaMemcpyAsync(b_sc.p, &h, sizeof h, cudaMemcpyHostToDevice, st));
  dt_gather_kernel<<<std::max(1, std::min(4 * ctx->num_sms, (N + 255) / 256)), 256, 0, st>>>(t, false);
  DCK(cudaGetLastError());
  DCK(cudaMemcpyAsync(vv.data(), b_vv.p, N * 4ull, cudaMemcpyDeviceToHost, st));
  DCK(cudaStreamSynchronize(st));
  if (vsum_after_reset) {
    long long sum = 0;
    for (int x = 0; x < N; ++x) sum += vv[x];
    *vsum_after_reset = sum;
  }
  return PPG_SUCCESS;
}

int ppg_run_pmbs_device(ppg_ctx* ctx, const double* root_poses, double* action_out, ppg_search_stats* stats,
                        char* sig_buf, int64_t sig_cap, int64_t* sig_len) {
  if (!ctx || !root_poses || !action_out) return PPG_EINVAL;
  if (!ctx->has_scene) {
    ctx->err = "no scene installed";
    return PPG_EINVAL;
  }
  if (ctx->group) return ppg::run_pmbs_sharded(ctx, root_poses, action_out, stats, sig_buf, sig_cap, sig_len);
  const auto t_start = std::chrono::steady_clock::now();
  const auto elapsed = [&t_start] {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
  };
  int rc = dt_begin(ctx, root_poses, false);
  if (rc != PPG_SUCCESS) return rc;
  const ppg_params& p = ctx->params;
  DTreeState& S = *ctx->dtree;
  cudaStream_t st = ctx->stream;
  const int n = S.n;
  const long long per_iter_actions = static_cast<long long>(p.n_envs) * n * S.na;
  DTScal h;
  std::memset(&h, 0, sizeof h);
  int stop = -1;
  const char* dbg = std::getenv("PPG_DTREE_DEBUG");
  const bool debug = dbg && dbg[0] == '1';
  const bool gdebug = dbg && dbg[0] == '2';  // graph mode, synchronize + check every launch
  bool regrown = false;
  // simulate hook (sharded driver): rollouts by the caller between the two
  // graphs of an iteration, per-pair rewards copied back as the harvest's bits
  const bool hooked = ctx->sim_hook != nullptr;
  int64_t hook_ctr[4] = {0, 0, 0, 0};
  std::vector<double> h_cp, h_rew;
  std::vector<int32_t> h_meta;
  const auto t_loop = std::chrono::steady_clock::now();
  for (;;) {
    // capacity for one more iteration (the host learns the sizes after each)
    {
      const int prev_it = h.iteration, prev_nodes = h.n_nodes;
      cudaError_t e = S.hsc ? cudaSuccess : cudaMallocHost(&S.hsc, sizeof(DTScal));
      if (e == cudaSuccess) e = cudaMemcpyAsync(S.hsc, S.t.sc, sizeof h, cudaMemcpyDeviceToHost, st);
      if (e == cudaSuccess) e = cudaStreamSynchronize(st);
      if (e == cudaSuccess) std::memcpy(&h, S.hsc, sizeof h);
      if (e != cudaSuccess) {
        char m[256];
        std::snprintf(m, sizeof m, "dtree: iteration after %d (nodes %d, cap %d, regrown %d): %s", prev_it,
                      prev_nodes, S.cap_nodes, regrown ? 1 : 0, cudaGetErrorString(e));
        ctx->err = m;
        return PPG_ECUDA;
      }
    }
    if (h.round_guard < 0) {
      ctx->err = "device tree: lockstep rounds exceeded the safety limit";
      return PPG_EINVAL;
    }
    if (h.async_ctl[3] != 0) {
      ctx->err = "device tree: asynchronous lockstep stalled (protocol error)";
      if (std::getenv("PPG_ASYNC_DUMP")) {  // protocol state at the stall (debugging)
        const int E = S.n_envs;
        std::vector<int32_t> ctr(static_cast<size_t>(kAsyncK) * kRingCtr), st(E), rd(E), nd(E), pu(E);
        std::vector<uint8_t> dn(E);
        cudaMemcpy(ctr.data(), S.l_actr.p, ctr.size() * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(st.data(), S.l_astate.p, E * 4ull, cudaMemcpyDeviceToHost);
        cudaMemcpy(rd.data(), S.l_around.p, E * 4ull, cudaMemcpyDeviceToHost);
        cudaMemcpy(nd.data(), S.l_node.p, E * 4ull, cudaMemcpyDeviceToHost);
        std::fprintf(stderr, "async stall: ctl");
        for (int k = 0; k < 16; ++k) std::fprintf(stderr, " %d", h.async_ctl[k]);
        std::fprintf(stderr, "\n");
        for (int k = 0; k < kAsyncK; ++k) {
          std::fprintf(stderr, " slot %d:", k);
          for (int j = 0; j < 10; ++j) std::fprintf(stderr, " %d", ctr[k * kRingCtr + j]);
          std::fprintf(stderr, "\n");
        }
        int cnt[8] = {};
        for (int e = 0; e < h.lock_dyn[1] && e < E; ++e) {
          const int v = st[e];
          cnt[v >= 0 && v < 7 ? v : 7]++;
          if (v != 2) std::fprintf(stderr, "  env %d state %d round %d node %d\n", e, v, rd[e], nd[e]);
        }
        std::fprintf(stderr, " states: ready %d await %d gone %d spec %d other %d\n", cnt[0], cnt[1], cnt[2], cnt[4],
                     cnt[7]);
      }
      return PPG_ECUDA;
    }
    if (h.err[0]) {
      char m[256];
      std::snprintf(m, sizeof m, "dtree: corrupt ancestor row: node %d depth %d ancestor %d (iteration %d, nodes %d)",
                    h.err[1], h.err[2], h.err[3], h.iteration, h.n_nodes);
      ctx->err = m;
      return PPG_EINVAL;
    }
    if (h.stop >= 0) {
      stop = h.stop;
      break;
    }
    if (!p.budget_iterations && h.iteration > 0 && elapsed() >= p.max_seconds) {
      stop = 0;
      break;
    }
    if (h.n_nodes + p.n_envs > S.cap_nodes || h.a_used + per_iter_actions > S.cap_actions) {
      const int want = std::max(2 * S.cap_nodes, h.n_nodes + p.n_envs);
      const long long wa = std::max(2 * S.cap_actions, h.a_used + per_iter_actions);
      if ((rc = dt_reserve(ctx, S, h.n_nodes, h.a_used, want, wa)) != PPG_SUCCESS) return rc;
      dt_views(ctx, S);
      regrown = true;
    }
    if (debug && !hooked) {
      if ((rc = dt_iteration_debug(ctx, S)) != PPG_SUCCESS) return rc;
      continue;
    }
    if (!S.exec && (rc = hooked ? dt_capture_hooked(ctx, S) : dt_capture(ctx, S)) != PPG_SUCCESS) {
      cudaStreamCaptureStatus cs;
      if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) {
        cudaGraph_t junk;
        cudaStreamEndCapture(st, &junk);
        if (junk) cudaGraphDestroy(junk);
      }
      cudaGetLastError();
      S.release_graph();
      return rc;
    }
    DCK(cudaGraphLaunch(S.exec, st));
    if (hooked) {
      DTScal hs;
      DCK(cudaMemcpyAsync(&hs, S.t.sc, sizeof hs, cudaMemcpyDeviceToHost, st));
      DCK(cudaStreamSynchronize(st));
      const int P = hs.n_pairs;
      if (P > 0) {
        h_cp.resize(static_cast<size_t>(P) * n * 3);
        h_meta.resize(static_cast<size_t>(P) * 3);
        h_rew.assign(P, 0.0);
        DCK(cudaMemcpyAsync(h_cp.data(), S.t.cp, h_cp.size() * 8, cudaMemcpyDeviceToHost, st));
        DCK(cudaMemcpyAsync(h_meta.data(), S.t.meta, h_meta.size() * 4, cudaMemcpyDeviceToHost, st));
        DCK(cudaStreamSynchronize(st));
        int64_t c4[4] = {0, 0, 0, 0};
        rc = ctx->sim_hook(ctx->sim_hook_user, h_cp.data(), h_meta.data(), P, p.n_envs, p.leaf_parallel, p.rng_seed,
                           static_cast<uint64_t>(hs.lock_dyn[3]), hs.lock_dyn[2], h_rew.data(), c4);
        if (rc != PPG_SUCCESS) {
          ctx->err = "simulate hook failed";
          return rc;
        }
        for (int k = 0; k < 4; ++k) hook_ctr[k] += c4[k];
        // backprop reads the rewards as the harvest's atomicMax bits
        DCK(cudaMemcpyAsync(S.la.rew, h_rew.data(), static_cast<size_t>(P) * 8, cudaMemcpyHostToDevice, st));
      }
      DCK(cudaGraphLaunch(S.exec_post, st));
    }
    if (gdebug) {
      const cudaError_t e = cudaStreamSynchronize(st);
      if (e != cudaSuccess) {
        char m[256];
        std::snprintf(m, sizeof m, "dtree graph debug: iteration %d (nodes %d, cap %d, regrown %d): %s", h.iteration,
                      h.n_nodes, S.cap_nodes, regrown ? 1 : 0, cudaGetErrorString(e));
        ctx->err = m;
        return PPG_ECUDA;
      }
    }
  }
  const double loop_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_loop).count();
  int64_t ctr[4];
  DCK(cudaMemcpyAsync(ctr, S.la.counters, 32, cudaMemcpyDeviceToHost, st));
  DCK(cudaStreamSynchronize(st));
  for (int k = 0; k < 4; ++k) ctr[k] += hook_ctr[k];
  return dt_finish(ctx, h, stop, elapsed(), loop_s, ctr, action_out, stats, sig_buf, sig_cap, sig_len);
}

}  // extern "C"
