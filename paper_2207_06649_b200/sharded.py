"""Multi-GPU batch_simulate: the lockstep engine (pmbs.cpp:133-205) sharded by
environment — the Python restatement of the exchange protocol that the
library runs natively (csrc/multi.cu, ppg_create_rank / ppg_create_multi),
used as the test double of that protocol on CPU (gloo, world_size 2) and
behind ppg_set_simulate_hook.

Each rank owns a contiguous range of global environment indices.  The
env -> node split and the RNG keys (pmbs.cpp:138-149, 211-213) use global
indices, so the union of the shards is the unsharded batch.  Environments
only interact through harvest_and_repurpose (pmbs.cpp:165-187): an env that
finishes by grasp moves to argmax_i W[i], W[i] = the remaining rollout work
of node i.  Within one pass the only change to W is W[best] += (>= 0), so
every re-purpose of the pass goes to the argmax of W at the start of the
pass.  That makes ONE exchange per lockstep round exact:

    report (device)   -> this shard's newly finished envs (rewards, grasp
                         flags) and W_local
    allreduce(sum)    -> W (the only collective of the round)
    harvest (local)   -> reward max per node; this shard's by-grasp envs go
                         to argmax W (strict >, W > 0, lowest node)
    repurpose (device)-> local envs restart at their new node
    step (device)     -> one round for the local active envs
    (loop while sum(W) > 0: a not-done env contributes cap - pushes >= 1)

Per-node rewards are a max, all-reduced once at the end.  `Comm` abstracts
the collectives: torch.distributed (NCCL on GPUs, gloo on CPU) or in-process
shards.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import List, Sequence

import numpy as np

from . import abi
from .abi import dptr, i64ptr, iptr, u8ptr


@dataclass
class Records:
    env: np.ndarray     # int32, increasing global env index
    node: np.ndarray    # int32
    grasp: np.ndarray   # uint8 finished by grasp
    reward: np.ndarray  # float64

    @staticmethod
    def empty() -> "Records":
        return Records(np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros(0, np.uint8), np.zeros(0, np.float64))

    @staticmethod
    def concat(parts: Sequence["Records"]) -> "Records":
        if not parts:
            return Records.empty()
        return Records(np.concatenate([p.env for p in parts]), np.concatenate([p.node for p in parts]),
                       np.concatenate([p.grasp for p in parts]), np.concatenate([p.reward for p in parts]))


def env_range(used: int, world: int, rank: int):
    """Contiguous, balanced split of global env indices [0, used)."""
    base, rem = divmod(used, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def best_node(W: np.ndarray) -> int:
    """argmax_i W[i] with strict > and W > 0, lowest node on ties (-1: none)
    — the reference's scan (pmbs.cpp:172-180) on the summed W."""
    if len(W) == 0:
        return -1
    b = int(np.argmax(W))
    return b if W[b] > 0 else -1


def harvest_local(rec: Records, best: int, leaf_parallel: bool, rewards: np.ndarray):
    """This shard's part of one harvest pass (pmbs.cpp:165-187): reward max of
    its newly finished envs; its by-grasp envs are re-purposed to `best` (the
    argmax of the GLOBAL W).  Returns the assignments (env, node)."""
    for k in range(len(rec.env)):
        nd = int(rec.node[k])
        r = float(rec.reward[k])
        if rewards[nd] < r:
            rewards[nd] = r
    if not leaf_parallel or best < 0:
        return np.zeros(0, np.int32), np.zeros(0, np.int32)
    env = rec.env[rec.grasp != 0].astype(np.int32)
    return env, np.full(len(env), best, np.int32)


class DeviceShard:
    """One shard of the lockstep batch on one ppg context (C-ABI ppg_lock_*)."""

    def __init__(self, ctx):
        self.ctx = ctx
        self.lib = ctx.lib

    def begin(self, node_poses, node_meta, n_nodes, used, lo, hi, leaf_parallel, seed, iteration, cap):
        self.lo, self.hi, self.n_nodes = lo, hi, n_nodes
        self._poses = np.ascontiguousarray(node_poses, np.float64)
        self._meta = np.ascontiguousarray(node_meta, np.int32)
        cap_e = max(1, hi - lo)
        self._env = np.zeros(cap_e, np.int32)
        self._node = np.zeros(cap_e, np.int32)
        self._grasp = np.zeros(cap_e, np.uint8)
        self._reward = np.zeros(cap_e, np.float64)
        self._W = np.zeros(n_nodes, np.int32)
        self.ctx._check(self.lib.ppg_lock_begin(self.ctx.ptr, dptr(self._poses), iptr(self._meta), n_nodes, used, lo,
                                                hi, int(leaf_parallel), seed & 0xFFFFFFFFFFFFFFFF, iteration, cap),
                        "ppg_lock_begin")

    def report(self):
        nrec, nact = ctypes.c_int32(), ctypes.c_int32()
        self.ctx._check(self.lib.ppg_lock_report(self.ctx.ptr, iptr(self._env), iptr(self._node), u8ptr(self._grasp),
                                                 dptr(self._reward), ctypes.byref(nrec), iptr(self._W),
                                                 ctypes.byref(nact)), "ppg_lock_report")
        k = nrec.value
        return (Records(self._env[:k].copy(), self._node[:k].copy(), self._grasp[:k].copy(), self._reward[:k].copy()),
                self._W.copy(), nact.value)

    def repurpose(self, env: np.ndarray, node: np.ndarray):
        env = np.ascontiguousarray(env, np.int32)
        node = np.ascontiguousarray(node, np.int32)
        if len(env):
            self.ctx._check(self.lib.ppg_lock_repurpose(self.ctx.ptr, iptr(env), iptr(node), len(env)),
                            "ppg_lock_repurpose")

    def step(self):
        self.ctx._check(self.lib.ppg_lock_step(self.ctx.ptr), "ppg_lock_step")

    def counters(self) -> np.ndarray:
        c = np.zeros(4, np.int64)
        self.ctx._check(self.lib.ppg_lock_counters(self.ctx.ptr, i64ptr(c)), "ppg_lock_counters")
        return c


class InProcessComm:
    """Several shards in this process (e.g. emulating ranks on one device)."""
    world = 1

    def gather_records(self, parts: List[Records]) -> Records:
        return Records.concat(parts)

    def sum(self, arr: np.ndarray) -> np.ndarray:
        return arr

    def sum_int(self, v: int) -> int:
        return v

    def max(self, arr: np.ndarray) -> np.ndarray:
        return arr


class TorchComm:
    """One shard per process; collectives over a torch.distributed group
    (NCCL between GPUs, gloo on CPU)."""

    def __init__(self, group=None, device=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.group = torch, dist, group
        self.world = dist.get_world_size(group)
        self.device = device if device is not None else torch.device("cpu")

    def _t(self, a):
        return self.torch.from_numpy(np.ascontiguousarray(a)).to(self.device)

    def gather_records(self, parts: List[Records]) -> Records:
        (mine,) = parts
        torch, dist = self.torch, self.dist
        n = self._t(np.array([len(mine.env)], np.int64))
        counts = [torch.zeros_like(n) for _ in range(self.world)]
        dist.all_gather(counts, n, group=self.group)
        counts = [int(c.item()) for c in counts]
        m = max(counts)
        if m == 0:
            return Records.empty()
        pad = np.zeros((m, 4), np.float64)  # env, node, grasp, reward as exact float64 payload
        k = len(mine.env)
        pad[:k, 0] = mine.env
        pad[:k, 1] = mine.node
        pad[:k, 2] = mine.grasp
        pad[:k, 3] = mine.reward
        t = self._t(pad)
        out = [torch.zeros_like(t) for _ in range(self.world)]
        dist.all_gather(out, t, group=self.group)
        rows = np.concatenate([o.cpu().numpy()[:c] for o, c in zip(out, counts)])
        return Records(rows[:, 0].astype(np.int32), rows[:, 1].astype(np.int32), rows[:, 2].astype(np.uint8),
                       np.ascontiguousarray(rows[:, 3]))

    def sum(self, arr: np.ndarray) -> np.ndarray:
        t = self._t(arr.astype(np.int64))
        self.dist.all_reduce(t, group=self.group)
        return t.cpu().numpy().astype(arr.dtype)

    def sum_int(self, v: int) -> int:
        return int(self.sum(np.array([v], np.int64))[0])

    def max(self, arr: np.ndarray) -> np.ndarray:
        """Element-wise max of non-negative float64 rewards (exact)."""
        t = self._t(arr.astype(np.float64))
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return t.cpu().numpy()


def sharded_simulate(shards, comm, node_poses, node_meta, n_envs: int, leaf_parallel: bool, seed: int,
                     iteration: int, depth_cap: int, ranges=None):
    """batch_simulate over the local `shards` (each with its global env range)
    of a batch sharded across `comm`: one W all-reduce per round, one reward
    max at the end.  Returns (rewards, counters)."""
    node_meta = np.ascontiguousarray(node_meta, np.int32)
    n_nodes = len(node_meta)
    used = n_envs if leaf_parallel else n_nodes
    if n_envs < n_nodes:
        raise ValueError("lockstep_simulate: fewer environments than nodes")
    for sh, (lo, hi) in zip(shards, ranges):
        sh.begin(node_poses, node_meta, n_nodes, used, lo, hi, leaf_parallel, seed, iteration, depth_cap)
    rewards = np.zeros(n_nodes, np.float64)
    rounds = 0
    while True:
        reps = [sh.report() for sh in shards]
        W = comm.sum(np.sum([r[1] for r in reps], axis=0).astype(np.int64))  # the round's one exchange
        best = best_node(W) if leaf_parallel else -1
        for sh, rep in zip(shards, reps):
            env, node = harvest_local(rep[0], best, leaf_parallel, rewards)
            sh.repurpose(env, node)
        if int(W.sum()) == 0:
            break
        for sh in shards:
            sh.step()
        rounds += 1
    rewards = comm.max(rewards)
    ctr = np.sum([sh.counters() for sh in shards], axis=0).astype(np.int64)
    ctr = comm.sum(ctr)
    ctr[1] = rounds
    return rewards, ctr


class ShardedSimulateHook:
    """Installs sharded_simulate as the planner's batch_simulate
    (ppg_set_simulate_hook), so ppg_run_pmbs on every rank runs the same tree
    (device-resident by default, dtree.cu) with the rollout batch sharded
    across ranks.  `extra_ctxs`: further local contexts that act as ranks
    rank+1, rank+2, ... (in-process emulation of a wider world on one GPU;
    their scene and parameters must match ctx's)."""

    def __init__(self, ctx, comm, world: int, rank: int, extra_ctxs=()):
        self.ctx, self.comm, self.world, self.rank = ctx, comm, world, rank
        self.shard = DeviceShard(ctx)
        self.shards = [self.shard] + [DeviceShard(c) for c in extra_ctxs]
        self.error = None

        def fn(user, node_poses, node_meta, n_nodes, n_envs, leaf_parallel, seed, iteration, depth_cap, rewards_out,
               counters):
            try:
                n = self.ctx._scene_table.n_objects
                poses = np.ctypeslib.as_array(node_poses, shape=(n_nodes, n, 3)).copy()
                meta = np.ctypeslib.as_array(node_meta, shape=(n_nodes, 3)).copy()
                used = n_envs if leaf_parallel else n_nodes
                rng = [env_range(used, self.world, self.rank + i) for i in range(len(self.shards))]
                r, c = sharded_simulate(self.shards, self.comm, poses, meta, n_envs, bool(leaf_parallel), seed,
                                        iteration, depth_cap, rng)
                np.ctypeslib.as_array(rewards_out, shape=(n_nodes,))[:] = r
                if counters:
                    np.ctypeslib.as_array(counters, shape=(4,))[:] = c
                return 0
            except Exception as e:  # surfaced by ppg_run_pmbs as an error
                self.error = e
                return abi.PPG_EINVAL

        self._fn = abi.SIMULATE_FN(fn)
        ctx.lib.ppg_set_simulate_hook(ctx.ptr, ctypes.cast(self._fn, ctypes.c_void_p), None)

    def remove(self):
        self.ctx.lib.ppg_set_simulate_hook(self.ctx.ptr, None, None)


def rank_context(device: int, params=None, group=None):
    """The library-native multi-GPU context of this process (one shard per
    rank under torchrun): rank 0 makes the NCCL id, torch.distributed
    broadcasts it, every rank creates ppg_create_rank over its own GPU.
    ppg_simulate / ppg_run_pmbs on it then shard the rollout batch with the
    per-round W all-reduce inside the library (csrc/multi.cu)."""
    import torch.distributed as dist

    from .api import Context, nccl_unique_id
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return Context.rank(device, rank, world, obj[0], params)
