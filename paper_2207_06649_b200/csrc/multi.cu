// multi.cu — multi-GPU sharding of the rollout batch (BASELINE
// configs[4]; north star item 4).
//
// The lockstep rollouts of one PMBS iteration (batch_simulate /
// lockstep_simulate, pmbs.cpp:133-234) partition by environment: shard r of G
// owns a contiguous range of the global env batch; env -> node split and RNG
// keys (seed, iteration, e) use GLOBAL env indices (lock_init_kernel), so the
// union of the shards is the unsharded batch.  The only interaction between
// environments is the sequential harvest (pmbs.cpp:165-187): an env that
// finished by grasp is re-purposed to argmax_i remaining_work(i).  During one
// pass the only change to W is W[best] += (>= 0), so every re-purpose of the
// pass goes to the SAME node — the argmax of W at the start of the pass.  So
// ONE exchange per round is exact: each shard computes its W (sum over its
// not-done envs), the shards' W are summed in place (NCCL all-reduce over
// NVLink), and every shard re-purposes its own envs to the argmax of the sum
// (lock_harvest_local_kernel / lock_harvest_apply_kernel).  The loop ends when
// the summed W is zero (no env active anywhere); per-node rewards are a max,
// all-reduced once at the end (bit patterns of non-negative doubles: uint64
// max).  The search tree itself is replicated (every shard runs the same
// select / expand / attach / backprop kernels on identical data), so no tree
// state moves between GPUs and the decision is bit-identical for any G.
//
// Transports:
//   NCCL   ppg_create_rank (one process per GPU, ncclCommInitRank with an id
//          from ppg_nccl_unique_id) or ppg_create_multi (one process, all
//          devices, ncclCommInitAll); libnccl is loaded at run time (dlopen:
//          the copy torch already loaded, else PPG_NCCL_LIB, else the system
//          libnccl.so.2), so the library has no link-time NCCL dependency.
//   LOCAL  ppg_create_multi(..., PPG_MULTI_EMULATE): G shards on ONE device
//          (tests): the exchange is one kernel over every shard's buffer,
//          ordered by events — no kernel ever waits on another.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "ctx_impl.cuh"

namespace ppg {

namespace {

struct NcclApi {
  void* h = nullptr;
  bool tried = false;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*commAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*commGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*getVersion)(int*) = nullptr;
};

NcclApi g_nccl;

template <class F>
bool sym(void* h, const char* name, F& f) {
  f = reinterpret_cast<F>(dlsym(h, name));
  return f != nullptr;
}

// Loads libnccl once: the copy already in the process (torch's) first, so
// one process never holds two NCCL builds.
const NcclApi* nccl() {
  if (g_nccl.tried) return g_nccl.h ? &g_nccl : nullptr;
  g_nccl.tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) {
    const char* p = std::getenv("PPG_NCCL_LIB");
    if (p) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
  }
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return nullptr;
  NcclApi& a = g_nccl;
  const bool ok = sym(h, "ncclGetUniqueId", a.getUniqueId) && sym(h, "ncclCommInitRank", a.commInitRank) &&
                  sym(h, "ncclCommInitAll", a.commInitAll) && sym(h, "ncclAllReduce", a.allReduce) &&
                  sym(h, "ncclGroupStart", a.groupStart) && sym(h, "ncclGroupEnd", a.groupEnd) &&
                  sym(h, "ncclCommDestroy", a.commDestroy) && sym(h, "ncclCommAbort", a.commAbort) &&
                  sym(h, "ncclCommGetAsyncError", a.commGetAsyncError) &&
                  sym(h, "ncclGetErrorString", a.getErrorString) && sym(h, "ncclGetVersion", a.getVersion);
  if (!ok) {
    dlclose(h);
    return nullptr;
  }
  a.h = h;
  return &a;
}

constexpr int kMaxLocalShards = 16;

struct LocalBufs {
  void* p[kMaxLocalShards];
  int n;
};

// LOCAL transport: every shard's buffer on one device; one kernel reduces
// element-wise over the shards and writes the result back to all of them.
__global__ void local_sum_i32_kernel(LocalBufs b, size_t count) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    int s = 0;
    for (int k = 0; k < b.n; ++k) s += static_cast<int32_t*>(b.p[k])[i];
    for (int k = 0; k < b.n; ++k) static_cast<int32_t*>(b.p[k])[i] = s;
  }
}

__global__ void local_sum_i64_kernel(LocalBufs b, size_t count) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    long long s = 0;
    for (int k = 0; k < b.n; ++k) s += static_cast<long long*>(b.p[k])[i];
    for (int k = 0; k < b.n; ++k) static_cast<long long*>(b.p[k])[i] = s;
  }
}

__global__ void local_max_u64_kernel(LocalBufs b, size_t count) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    unsigned long long m = 0;
    for (int k = 0; k < b.n; ++k) m = max(m, static_cast<unsigned long long*>(b.p[k])[i]);
    for (int k = 0; k < b.n; ++k) static_cast<unsigned long long*>(b.p[k])[i] = m;
  }
}

}  // namespace

struct Group {
  enum Kind { kNccl = 1, kLocal = 2 } kind = kNccl;
  int rank0 = 0, world = 1;
  std::vector<ppg_ctx*> m;          // m[0] is the context the caller holds
  std::vector<ncclComm_t> comms;    // NCCL: one per member
  std::vector<cudaEvent_t> ev;      // LOCAL: per member
  cudaEvent_t ev_done = nullptr;    // LOCAL: the reduction finished
  bool aborted = false;
};

int group_size(const Group* g) { return static_cast<int>(g->m.size()); }
ppg_ctx* group_member(const Group* g, int k) { return g->m[k]; }
int group_rank0(const Group* g) { return g->rank0; }
int group_world(const Group* g) { return g->world; }

namespace {

int nccl_fail(ppg_ctx* ectx, const char* what, ncclResult_t r) {
  const NcclApi* a = nccl();
  ectx->err = std::string(what) + ": " + (a ? a->getErrorString(r) : "NCCL unavailable");
  return PPG_ECUDA;
}

template <class K>
int local_reduce(ppg_ctx* ectx, Group* g, void* const* bufs, size_t count, K kernel) {
  LocalBufs b{};
  b.n = static_cast<int>(g->m.size());
  for (int k = 0; k < b.n; ++k) b.p[k] = bufs[k];
  cudaStream_t s0 = g->m[0]->stream;
  for (int k = 1; k < b.n; ++k) {
    if (cudaEventRecord(g->ev[k], g->m[k]->stream) != cudaSuccess ||
        cudaStreamWaitEvent(s0, g->ev[k], 0) != cudaSuccess) {
      ectx->err = "local exchange: event ordering failed";
      return PPG_ECUDA;
    }
  }
  const int grid = static_cast<int>(std::min<size_t>(1184, (count + 255) / 256 + 1));
  kernel<<<grid, 256, 0, s0>>>(b, count);
  if (cudaGetLastError() != cudaSuccess || cudaEventRecord(g->ev_done, s0) != cudaSuccess) {
    ectx->err = "local exchange: launch failed";
    return PPG_ECUDA;
  }
  for (int k = 1; k < b.n; ++k)
    if (cudaStreamWaitEvent(g->m[k]->stream, g->ev_done, 0) != cudaSuccess) {
      ectx->err = "local exchange: event ordering failed";
      return PPG_ECUDA;
    }
  return PPG_SUCCESS;
}

int nccl_reduce(ppg_ctx* ectx, Group* g, void* const* bufs, size_t count, ncclDataType_t dt, ncclRedOp_t op) {
  const NcclApi* a = nccl();
  if (!a) {
    ectx->err = "NCCL unavailable";
    return PPG_ECUDA;
  }
  const bool grouped = g->m.size() > 1;
  ncclResult_t r = ncclSuccess;
  if (grouped && (r = a->groupStart()) != ncclSuccess) return nccl_fail(ectx, "ncclGroupStart", r);
  for (size_t k = 0; k < g->m.size(); ++k) {
    cudaSetDevice(g->m[k]->device);
    r = a->allReduce(bufs[k], bufs[k], count, dt, op, g->comms[k], g->m[k]->stream);
    if (r != ncclSuccess) {
      if (grouped) a->groupEnd();
      return nccl_fail(ectx, "ncclAllReduce", r);
    }
  }
  if (grouped && (r = a->groupEnd()) != ncclSuccess) return nccl_fail(ectx, "ncclGroupEnd", r);
  return PPG_SUCCESS;
}

}  // namespace

int group_allreduce_sum_i32(ppg_ctx* ectx, Group* g, int32_t* const* bufs, size_t count) {
  if (count == 0) return PPG_SUCCESS;
  if (g->kind == Group::kLocal)
    return local_reduce(ectx, g, reinterpret_cast<void* const*>(bufs), count, local_sum_i32_kernel);
  return nccl_reduce(ectx, g, reinterpret_cast<void* const*>(bufs), count, ncclInt32, ncclSum);
}

int group_allreduce_sum_i64(ppg_ctx* ectx, Group* g, long long* const* bufs, size_t count) {
  if (count == 0) return PPG_SUCCESS;
  if (g->kind == Group::kLocal)
    return local_reduce(ectx, g, reinterpret_cast<void* const*>(bufs), count, local_sum_i64_kernel);
  return nccl_reduce(ectx, g, reinterpret_cast<void* const*>(bufs), count, ncclInt64, ncclSum);
}

int group_allreduce_max_u64(ppg_ctx* ectx, Group* g, unsigned long long* const* bufs, size_t count) {
  if (count == 0) return PPG_SUCCESS;
  if (g->kind == Group::kLocal)
    return local_reduce(ectx, g, reinterpret_cast<void* const*>(bufs), count, local_max_u64_kernel);
  return nccl_reduce(ectx, g, reinterpret_cast<void* const*>(bufs), count, ncclUint64, ncclMax);
}

int group_wait(ppg_ctx* ectx, Group* g) {
  static const double timeout = [] {
    const char* v = std::getenv("PPG_NCCL_TIMEOUT_S");
    return v ? std::atof(v) : 300.0;
  }();
  const auto t0 = std::chrono::steady_clock::now();
  const NcclApi* a = g->kind == Group::kNccl ? nccl() : nullptr;
  for (size_t k = 0; k < g->m.size(); ++k) {
    cudaSetDevice(g->m[k]->device);
    int spins = 0;
    for (;;) {
      const cudaError_t e = cudaStreamQuery(g->m[k]->stream);
      if (e == cudaSuccess) break;
      if (e != cudaErrorNotReady) {
        ectx->err = std::string("shard ") + std::to_string(g->rank0 + k) + ": " + cudaGetErrorString(e);
        return PPG_ECUDA;
      }
      if (a) {
        ncclResult_t ar = ncclSuccess;
        a->commGetAsyncError(g->comms[k], &ar);
        if (ar != ncclSuccess && ar != ncclInProgress) return nccl_fail(ectx, "NCCL async error", ar);
      }
      if (++spins > 64) {
        std::this_thread::sleep_for(std::chrono::microseconds(5));
        if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout) {
          if (a && !g->aborted) {
            for (ncclComm_t c : g->comms) a->commAbort(c);
            g->comms.assign(g->comms.size(), nullptr);
            g->aborted = true;
          }
          ectx->err = "multi-GPU exchange timed out (PPG_NCCL_TIMEOUT_S); communicators aborted";
          return PPG_ECUDA;
        }
      }
    }
  }
  return PPG_SUCCESS;
}

void group_destroy(ppg_ctx* ctx) {
  Group* g = ctx->group;
  if (!g) return;
  ctx->group = nullptr;
  const NcclApi* a = g->kind == Group::kNccl ? nccl() : nullptr;
  for (size_t k = 0; k < g->m.size(); ++k) {
    cudaSetDevice(g->m[k]->device);
    if (g->m[k]->stream) cudaStreamSynchronize(g->m[k]->stream);
    if (a && k < g->comms.size() && g->comms[k]) a->commDestroy(g->comms[k]);
    if (k < g->ev.size() && g->ev[k]) cudaEventDestroy(g->ev[k]);
  }
  if (g->ev_done) cudaEventDestroy(g->ev_done);
  for (size_t k = 1; k < g->m.size(); ++k) {
    g->m[k]->group = nullptr;
    ppg_destroy(g->m[k]);
  }
  delete g;
}

// ---------------------------------------------------------------------------
// sharded batch_simulate (ppg_simulate on a multi-GPU context)

namespace {

int ensure_go(ppg_ctx* c) {
  if (c->l_go.ensure(16) != cudaSuccess) return PPG_ECUDA;
  if (!c->h_go && cudaMallocHost(&c->h_go, 16) != cudaSuccess) return PPG_ECUDA;
  return PPG_SUCCESS;
}

}  // namespace

bool shard_waves_enabled(const ppg_ctx* ctx) {
  static const bool on = [] {
    const char* v = std::getenv("PPG_SHARD_WAVES");
    return !(v && v[0] == '0');
  }();
  // the wave physics is the lane-per-env disc kernel
  return on && wave_enabled(ctx) && ctx->scene_all_discs && ctx->scene.n <= kDiscMaxN && ctx->disc_kernels &&
         !ctx->warp_max_explicit;
}

// Wave rounds over shards (warp_env.cu): per wave every shard packs its W ring
// and per-round (arrived, gone) counts, ONE all-reduce sums them, and every
// shard's harvest decides / completes rounds from the identical sums (so all
// shards take the same decisions and stop at the same wave) while applying
// the decisions to its own envs; then sample, budgeted physics, post.  No
// hand-over to the asynchronous kernel (its exchange would be continuous).
int sharded_wave_rounds(ppg_ctx* ctx, Group* g, std::vector<ShardWave>& sw, int P, int work) {
  const int M = static_cast<int>(sw.size());
  // W ring, per-round (arrived, gone), then the pending bounds of the next
  // undecided round (round, near count, per node) — warp_env.cu wave_pack_kernel
  const size_t count = static_cast<size_t>(kAsyncK) * P + 2 * kAsyncK + 2 + P;
  std::vector<int32_t*> gb(M);
  for (int k = 0; k < M; ++k) {
    ppg_ctx* c = sw[k].c;
    CK(cudaSetDevice(c->device));
    CK(c->l_gring.ensure(count * sizeof(int32_t)));
    LockArgs& a = sw[k].la;
    gb[k] = a.g_ring = c->l_gring.as<int32_t>();
    a.round_mode = nullptr;
    a.cond = 0;
    a.go = a.a_ctl + 7;
    a.wave_switch = 0;  // never hand over
    a.wave_budget = c->wave_budget;
  }
  const int pack_grid = static_cast<int>(std::min<size_t>((count + 255) / 256, 1024));
  for (int wave = 0;; ++wave) {
    for (int k = 0; k < M; ++k) {
      ppg_ctx* c = sw[k].c;
      CK(cudaSetDevice(c->device));
      wave_pack_kernel<<<pack_grid, 256, 0, c->stream>>>(sw[k].la);
      wave_pack_pending_kernel<<<std::max(1, std::min(4 * c->num_sms, (work + 255) / 256)), 256, 0, c->stream>>>(sw[k].la);
      CK(cudaGetLastError());
    }
    int rc = group_allreduce_sum_i32(ctx, g, gb.data(), count);
    if (rc != PPG_SUCCESS) return rc;
    for (int k = 0; k < M; ++k) {
      ppg_ctx* c = sw[k].c;
      CK(cudaSetDevice(c->device));
      if ((rc = launch_wave(c, *sw[k].C, sw[k].la, sw[k].ra, work, c->stream)) != PPG_SUCCESS) {
        ctx->err = c->err;
        return rc;
      }
      CK(cudaMemcpyAsync(c->h_go, sw[k].la.a_ctl + 7, 4, cudaMemcpyDeviceToHost, c->stream));
    }
    if ((rc = group_wait(ctx, g)) != PPG_SUCCESS) return rc;
    const int go = sw[0].c->h_go[0];
    for (int k = 1; k < M; ++k)
      if (sw[k].c->h_go[0] != go) {
        ctx->err = "sharded wave rounds: shards disagree on termination";
        return PPG_EINVAL;
      }
    if (!go) return PPG_SUCCESS;
    if (wave > 4 * kLockRoundLimit) {
      ctx->err = "sharded wave rounds did not terminate";
      return PPG_EINVAL;
    }
  }
}

int simulate_sharded(ppg_ctx* ctx, const double* node_poses, const int32_t* node_meta, int n_nodes, int n_envs,
                     int leaf_parallel, uint64_t seed, uint64_t iteration, int depth_cap, double* rewards_out,
                     int64_t* counters) {
  Group* g = ctx->group;
  const int M = group_size(g), G = g->world;
  const int used = leaf_parallel ? n_envs : n_nodes;
  for (int k = 0; k < M; ++k) {
    ppg_ctx* c = g->m[k];
    int rc = lock_check(c, n_nodes, n_envs, depth_cap);
    if (rc != PPG_SUCCESS) {
      ctx->err = c->err;
      return rc;
    }
    CK(cudaSetDevice(c->device));
    const int r = g->rank0 + k;
    const int lo = static_cast<int>(static_cast<long long>(used) * r / G);
    const int hi = static_cast<int>(static_cast<long long>(used) * (r + 1) / G);
    rc = lock_setup(c, node_poses, node_meta, n_nodes, hi - lo, used, lo, leaf_parallel, seed, iteration, depth_cap);
    if (rc == PPG_SUCCESS) rc = ensure_go(c);
    if (rc != PPG_SUCCESS) {
      ctx->err = c->err.empty() ? "sharded simulate: setup failed" : c->err;
      return rc;
    }
    c->la.go = c->l_go.as<int32_t>();
    c->lock_active_hint = hi - lo;
  }
  bool waves = true;
  for (int k = 0; k < M; ++k) waves = waves && shard_waves_enabled(g->m[k]);
  std::vector<int32_t*> wb(M);
  std::vector<unsigned long long*> rb(M);
  std::vector<long long*> cb(M);
  for (int k = 0; k < M; ++k) {
    wb[k] = g->m[k]->la.W;
    rb[k] = g->m[k]->la.rew;
    cb[k] = g->m[k]->la.counters;
  }
  for (;;) {
    // one harvest pass: local W -> exchange (sum) -> apply with the global W
    for (int k = 0; k < M; ++k) {
      ppg_ctx* c = g->m[k];
      CK(cudaSetDevice(c->device));
      lock_harvest_local_kernel<<<1, 1024, 0, c->stream>>>(c->lc, c->la);
      CK(cudaGetLastError());
    }
    int rc = group_allreduce_sum_i32(ctx, g, wb.data(), static_cast<size_t>(n_nodes));
    if (rc != PPG_SUCCESS) return rc;
    for (int k = 0; k < M; ++k) {
      ppg_ctx* c = g->m[k];
      CK(cudaSetDevice(c->device));
      lock_harvest_apply_kernel<<<1, 1024, 0, c->stream>>>(c->lc, c->la);
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(c->h_go, c->la.go, 4, cudaMemcpyDeviceToHost, c->stream));
      CK(cudaMemcpyAsync(c->h_go + 1, c->la.n_active, 4, cudaMemcpyDeviceToHost, c->stream));
    }
    if ((rc = group_wait(ctx, g)) != PPG_SUCCESS) return rc;
    const int go = g->m[0]->h_go[0];
    for (int k = 1; k < M; ++k)
      if (g->m[k]->h_go[0] != go) {
        ctx->err = "sharded simulate: shards disagree on termination";
        return PPG_EINVAL;
      }
    if (!go) break;
    if (waves) {  // every remaining round as waves, one exchange per wave
      std::vector<ShardWave> sw(M);
      for (int k = 0; k < M; ++k) sw[k] = ShardWave{g->m[k], &g->m[k]->lc, g->m[k]->la, g->m[k]->lra};
      const int work = (used + G - 1) / G;
      if ((rc = sharded_wave_rounds(ctx, g, sw, n_nodes, work)) != PPG_SUCCESS) return rc;
      break;
    }
    for (int k = 0; k < M; ++k) {
      ppg_ctx* c = g->m[k];
      CK(cudaSetDevice(c->device));
      const int act = c->h_go[1];
      if (act > 0 && (rc = lock_round(c, act)) != PPG_SUCCESS) {
        ctx->err = c->err;
        return rc;
      }
    }
  }
  int rc = group_allreduce_max_u64(ctx, g, rb.data(), static_cast<size_t>(n_nodes));
  if (rc == PPG_SUCCESS) rc = group_allreduce_sum_i64(ctx, g, cb.data(), 4);
  if (rc != PPG_SUCCESS) return rc;
  ppg_ctx* c0 = g->m[0];
  CK(cudaSetDevice(c0->device));
  CK(cudaMemcpyAsync(rewards_out, c0->la.rew, static_cast<size_t>(n_nodes) * 8, cudaMemcpyDeviceToHost, c0->stream));
  int64_t ctr[4];
  CK(cudaMemcpyAsync(ctr, c0->la.counters, 32, cudaMemcpyDeviceToHost, c0->stream));
  if ((rc = group_wait(ctx, g)) != PPG_SUCCESS) return rc;
  if (counters) {
    counters[0] = ctr[0];
    counters[1] = ctr[1] / G;  // every shard counts every round
    counters[2] = ctr[2];
    counters[3] = ctr[3];
  }
  return PPG_SUCCESS;
}

}  // namespace ppg

// ---------------------------------------------------------------------------
// C-ABI

extern "C" {

int ppg_nccl_unique_id(uint8_t* id) {
  if (!id) return PPG_EINVAL;
  const ppg::NcclApi* a = ppg::nccl();
  if (!a) return PPG_ECUDA;
  ncclUniqueId u;
  if (a->getUniqueId(&u) != ncclSuccess) return PPG_ECUDA;
  std::memcpy(id, &u, sizeof u);
  return PPG_SUCCESS;
}

ppg_ctx* ppg_create_rank(int device, int rank, int world, const uint8_t* nccl_id, const ppg_params* params,
                         int* err) {
  if (err) *err = PPG_SUCCESS;
  if (world < 1 || rank < 0 || rank >= world || (world > 1 && !nccl_id)) {
    if (err) *err = PPG_EINVAL;
    return nullptr;
  }
  ppg_ctx* ctx = ppg_create(device, params, err);
  if (!ctx) return nullptr;
  auto* g = new ppg::Group;
  g->kind = ppg::Group::kNccl;
  g->rank0 = rank;
  g->world = world;
  g->m = {ctx};
  g->comms.assign(1, nullptr);
  ctx->group = g;
  const ppg::NcclApi* a = ppg::nccl();
  ncclUniqueId u;
  if (world == 1) {
    if (a && a->getUniqueId(&u) != ncclSuccess) a = nullptr;
  } else {
    std::memcpy(&u, nccl_id, sizeof u);
  }
  if (!a || (cudaSetDevice(device), a->commInitRank(&g->comms[0], world, u, rank)) != ncclSuccess) {
    if (err) *err = PPG_ECUDA;
    ppg_destroy(ctx);
    return nullptr;
  }
  return ctx;
}

ppg_ctx* ppg_create_multi(const int* devices, int n_dev, int flags, const ppg_params* params, int* err) {
  if (err) *err = PPG_SUCCESS;
  if (!devices || n_dev < 1 || n_dev > ppg::kMaxLocalShards) {
    if (err) *err = PPG_EINVAL;
    return nullptr;
  }
  const bool emulate = (flags & PPG_MULTI_EMULATE) != 0;
  if (emulate)
    for (int k = 1; k < n_dev; ++k)
      if (devices[k] != devices[0]) {
        if (err) *err = PPG_EINVAL;  // emulated shards share one device
        return nullptr;
      }
  std::vector<ppg_ctx*> m;
  for (int k = 0; k < n_dev; ++k) {
    ppg_ctx* c = ppg_create(devices[k], params, err);
    if (!c) {
      for (ppg_ctx* x : m) ppg_destroy(x);
      return nullptr;
    }
    m.push_back(c);
  }
  auto* g = new ppg::Group;
  g->kind = emulate ? ppg::Group::kLocal : ppg::Group::kNccl;
  g->rank0 = 0;
  g->world = n_dev;
  g->m = m;
  for (ppg_ctx* c : m) c->group = g;  // members know the group (destroy goes through m[0])
  bool ok = true;
  if (emulate) {
    g->ev.assign(n_dev, nullptr);
    cudaSetDevice(devices[0]);
    for (int k = 0; k < n_dev && ok; ++k) ok = cudaEventCreateWithFlags(&g->ev[k], cudaEventDisableTiming) == cudaSuccess;
    ok = ok && cudaEventCreateWithFlags(&g->ev_done, cudaEventDisableTiming) == cudaSuccess;
  } else {
    const ppg::NcclApi* a = ppg::nccl();
    g->comms.assign(n_dev, nullptr);
    ok = a && a->commInitAll(g->comms.data(), n_dev, devices) == ncclSuccess;
  }
  if (!ok) {
    if (err) *err = PPG_ECUDA;
    ppg_destroy(m[0]);
    return nullptr;
  }
  return m[0];
}

int ppg_shard_info(ppg_ctx* ctx, int* rank, int* world, int* shards_here, int* transport) {
  if (!ctx) return PPG_EINVAL;
  const ppg::Group* g = ctx->group;
  if (rank) *rank = g ? g->rank0 : 0;
  if (world) *world = g ? g->world : 1;
  if (shards_here) *shards_here = g ? static_cast<int>(g->m.size()) : 1;
  if (transport) *transport = !g ? 0 : g->kind == ppg::Group::kNccl ? 1 : 2;
  return PPG_SUCCESS;
}

}  // extern "C"
