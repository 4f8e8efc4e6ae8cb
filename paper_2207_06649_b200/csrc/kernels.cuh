// kernels.cuh — kernel argument blocks shared by the kernels (kernels.cu) and
// the host context (ctx.cu).
#pragma once

#include <cstdint>

#include "physics.cuh"

namespace ppg {

struct ShapesDev {
  int* kind = nullptr;      // [n][T]
  double* rad = nullptr;    // [n][T]
  double* br = nullptr;     // [n][T]
  int* nv = nullptr;        // [n][T]
  double* verts = nullptr;  // [T][n][kMaxV][2]
  int* target = nullptr;    // [T]
  int T = 0;
  int n = 0;
  int capT = 0;
  __host__ __device__ ShapeView view(int t) const { return ShapeView{kind, rad, br, nv, verts, T, t, n}; }
};

struct ResolveArgs {
  ShapesDev S;
  const double* poses_in;  // [E][n][3]
  const double* pushes;    // [E][4]
  double* poses_out;       // [E][n][3]
  int32_t* status;         // [E]
  double* residual;        // [E] or null
  long long* counts;       // [E][8] (counting variant)
  int E;
  const int* idx = nullptr;    // optional env-slot indirection (lockstep / expand)
  const int* E_dev = nullptr;  // optional device-side count (overrides E)
  int* work_counter = nullptr; // resolve_warp_kernel: persistent warps take envs from this counter
  // streamed host batches (resolve_disc_kernel): inputs arrive slice by slice
  // while the kernel runs; slice k = env / slice_envs
  const unsigned* ready = nullptr;  // [slices]: == epoch once slice k's inputs are resident
  unsigned* done = nullptr;         // [slices]: finished envs (the copy-back stream waits on it)
  unsigned epoch = 0;
  int slice_envs = 0;
  bool rad_env_major = false;       // S.rad in the host layout [E][n] instead of [n][T]
  // poses_out / status / residual are mapped pinned HOST memory: each
  // finished env's poses leave in one warp-coalesced write (no copy-back)
  bool zc_out = false;
  // wave rounds (rollouts, resolve_disc_kernel<N, true>): an env runs at most
  // `budget` projection iterations per launch; an unfinished one yields
  // (positions in place, progress (step << 8 | iter, active mask) saved,
  // status 3) and resumes in the next launch; finished envs are appended
  // to fin_list.  resume_si[e] < 0: a fresh push.
  int32_t* resume_si = nullptr;
  uint32_t* resume_active = nullptr;
  int32_t* fin_list = nullptr;
  int32_t* fin_count = nullptr;
  int budget = 0;
  const int* budget_dev = nullptr;  // if set, the budget is read on the device (the graph's last wave: unbounded)
};

struct SampleArgs {
  ShapesDev S;
  const double* poses;  // [E][n][3]
  double* out;          // [E][n*na][4]
  int32_t* count;       // [E]
  uint8_t* grasp;       // [E] (grasp kernel)
  double* margin;       // [E]
  double* bx;           // [E]
  double* by;           // [E]
  int32_t* bk;          // [E]
  int E;
};

struct ExpandArgs {
  ShapesDev S;
  const double* parent_poses;  // [P][n][3]
  const double* actions;       // [P][4]
  double* child_poses;         // [P][n][3]
  int32_t* status;             // [P]
  uint8_t* grasp;              // [P]
  int32_t* n_untried;          // [P]
  double* untried;             // [P][n*na][4]
  int P;
  const int* P_dev = nullptr;  // optional device-side count (overrides P; device tree)
};

// Lockstep engine state (pmbs.cpp:133-205), all in HBM.
struct LockArgs {
  ShapesDev S;
  const double* node_poses;  // [n_nodes][n][3]
  const int32_t* node_meta;  // [n_nodes][3] depth, graspable, dead
  int n_nodes;
  int used;       // environments in use on this shard (local slots 0..used-1)
  int used_global = 0;  // environments of the whole batch (env -> node split, RNG keys)
  int env_lo = 0;       // global index of local slot 0 (sharded lockstep)
  int leaf_parallel;
  int cap;        // depth cap d_T + d_s
  uint64_t seed, iteration;
  // per-env
  int32_t* env_node;
  int32_t* env_pushes;
  uint8_t* env_done;
  uint8_t* env_bygrasp;
  uint8_t* env_harvested;
  uint8_t* env_flag;
  double* env_reward;
  double* env_poses;    // [E][n][3] (the physics kernels' AoS layout)
  double* env_push;     // [E][4] this round's push
  int32_t* env_status;  // [E] this round's resolve status
  int32_t* stepping;    // [used] envs with a push this round (disc pipeline)
  int32_t* n_stepping;  // [1]
  // sharded-lockstep report records (global env, node, by_grasp, reward)
  int32_t* rec_env = nullptr;
  int32_t* rec_node = nullptr;
  uint8_t* rec_grasp = nullptr;
  double* rec_reward = nullptr;
  int32_t* n_rec = nullptr;
  uint64_t* mt;         // [312][E]
  int32_t* mt_idx;      // [E]
  int E;                // allocated stride for env arrays
  // per-node
  int32_t* W;                // [n_nodes] remaining work
  unsigned long long* rew;   // [n_nodes] max reward bits (rewards >= 0)
  // round bookkeeping
  int32_t* active;           // [used]
  int32_t* n_active;         // [1]
  long long* counters;       // [4] steps, rounds, repurposes, resolve calls
  // device tree (dtree.cu): per-iteration values read on the device, so one
  // captured graph serves every PMBS iteration
  const int32_t* dyn = nullptr;        // [6] n_nodes, used, depth cap, iteration, seed lo, seed hi (overrides)
  unsigned long long cond = 0;         // graph WHILE handle: harvest sets it to (n_active > 0)
  // adaptive rounds (device tree): harvest writes *round_mode = 1 (hybrid:
  // warp sampler + lane physics) when n_active >= hybrid_min, else 0 (one
  // warp per env); the kernels of the other mode return at once
  int* round_mode = nullptr;
  int hybrid_min = 0;
  // device tree: rounds of the current lockstep call; the harvest stops the
  // WHILE loop (and marks the counter negative) past kLockRoundLimit, so a
  // bug surfaces as an error instead of a hung graph
  int* round_guard = nullptr;
  // sharded lockstep (multi-GPU, multi.cu): shard shard_r of shard_g owns a
  // contiguous range of the global env batch (with `dyn`, the range follows
  // the iteration's used-env count on the device).  The harvest is split
  // around ONE exchange per round: lock_harvest_local_kernel writes this
  // shard's W, the exchange sums W over the shards in place, and
  // lock_harvest_apply_kernel re-purposes with the global W and writes `go`
  // (any environment active anywhere) for the host.
  int shard_r = 0, shard_g = 1;
  int32_t* go = nullptr;
  // asynchronous lockstep (warp_env.cu lock_async_kernel): per env its
  // completed rounds and state (0 runnable, 1 awaiting the harvest of its
  // round, 2 gone, 3 + node: re-purposed to node, not yet applied); a ring
  // of kAsyncK rounds: W [K][a_wcap], counters [K][4] (arrived, gone at this
  // round, done-list length, -), done lists [K][E]; control [8] (harvested
  // round H, finished, gone so far, error, wave set up, switch to
  // asynchronous, host round-mode word, host go word, wave budget)
  int32_t* env_round = nullptr;
  int32_t* env_state = nullptr;
  int32_t* a_W = nullptr;
  int32_t* a_ctr = nullptr;
  int32_t* a_dl = nullptr;
  int32_t* a_ctl = nullptr;
  // sharded wave rounds (multi.cu / dtree.cu): every shard's W ring [K][n_nodes]
  // and (arrived, gone) per ring slot [K][2], summed over the shards before
  // each wave's harvest, which decides and completes rounds from these sums
  int32_t* g_ring = nullptr;
  // asynchronous lockstep: per ring slot, per node, the most the envs that will
  // step that round but have not finished it can still add to W [K][a_wcap]
  // (count of those envs: ring slot field [6])
  int32_t* a_P = nullptr;
  // speculative re-purposing: per env (node, pushes before, saved mt_idx, resolve counted)
  int4* a_spec = nullptr;
  int a_wcap = 0;
  // wave rounds (warp_env.cu wave_*_kernel): envs whose physics finished in
  // this wave (post pending), and the resumable physics progress
  int32_t* fin_list = nullptr;
  int32_t* fin_count = nullptr;
  int32_t* resume_si = nullptr;
  uint32_t* resume_active = nullptr;
  int wave_switch = 0;   // in-flight env-steps below which the waves hand over to the asynchronous kernel
  int wave_budget = 0;   // projection iterations per env per wave
  // PPG_STEP_TRACE (experiments): one record per latency-mode env-step
  // {env, round, start/end globaltimer ns, flags} appended at step_trace[1 + k]
  unsigned long long* step_trace = nullptr;
};

constexpr int kLockRoundLimit = 1 << 20;
#ifndef PPG_ASYNC_K
#define PPG_ASYNC_K 16
#endif
constexpr int kAsyncK = PPG_ASYNC_K;  // ring depth: rounds an env may run ahead of the last complete round
constexpr int kRingCtr = 16;  // ints per ring slot: arrived, gone at this round, done-list length, decided round,
                              // decision, applied, near count, -, provisional decision (u64 at [8])

// Applies the device-side per-iteration overrides (device tree mode).
__device__ __forceinline__ void lock_dyn(LockArgs& a) {
  if (a.dyn) {
    a.n_nodes = a.dyn[0];
    a.used = a.dyn[1];
    a.used_global = a.dyn[1];
    if (a.shard_g > 1) {  // this shard's contiguous part of the global batch
      const long long ug = a.dyn[1];
      const int lo = static_cast<int>(ug * a.shard_r / a.shard_g);
      const int hi = static_cast<int>(ug * (a.shard_r + 1) / a.shard_g);
      a.env_lo = lo;
      a.used = hi - lo;
    }
    a.cap = a.dyn[2];
    a.iteration = static_cast<uint64_t>(static_cast<uint32_t>(a.dyn[3]));
    a.seed = static_cast<uint64_t>(static_cast<uint32_t>(a.dyn[4])) |
             static_cast<uint64_t>(static_cast<uint32_t>(a.dyn[5])) << 32;
  }
}

// RolloutCursor ctor (mcts.cpp:121-140) for env e at node `node`.
PPG_DI void cursor_init(const SimConst& C, const LockArgs& a, int e, int node) {
  const int32_t* m = a.node_meta + node * 3;
  const int depth = m[0];
  a.env_node[e] = node;
  a.env_pushes[e] = depth;
  uint8_t done = 0, byg = 0;
  double reward = 0.0;
  if (m[1]) {
    done = 1;
    byg = 1;
    reward = C.gamma_pow[depth];
  } else if (m[2]) {
    done = 1;
  } else if (depth >= a.cap) {
    done = 1;
  }
  a.env_done[e] = done;
  a.env_bygrasp[e] = byg;
  a.env_reward[e] = reward;
  const int n = C.n;
  const double* src = a.node_poses + static_cast<size_t>(node) * n * 3;
  double* dst = a.env_poses + static_cast<size_t>(e) * n * 3;
  for (int i = 0; i < 3 * n; ++i) dst[i] = src[i];
}

}  // namespace ppg
