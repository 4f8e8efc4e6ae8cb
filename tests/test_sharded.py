"""Multi-GPU lockstep sharding (paper_2207_06649_b200.sharded) on CPU: the
host-side exchange + harvest logic with scripted rollout tasks — the
reference's own fake backend (ScriptedTask, test_pmbs.cpp:42-56) — against
a literal restatement of lockstep_simulate (pmbs.cpp:133-205), in-process
and across 2 gloo ranks (world_size 2)."""
import os
import socket
from dataclasses import dataclass

import numpy as np
import pytest

from paper_2207_06649_b200.sharded import InProcessComm, Records, env_range, sharded_simulate


@dataclass
class Script:
    steps: int
    reward: float
    by_grasp: bool


def lockstep_reference(n_nodes, n_envs, leaf_parallel, factory):
    """pmbs.cpp:133-205, restated literally (test oracle)."""
    used = n_envs if leaf_parallel else n_nodes
    env_node = []
    base, rem = divmod(used, n_nodes)
    for i in range(n_nodes):
        env_node += [i] * (base + (1 if i < rem else 0))
    calls = []
    left, tasks = [0] * used, [None] * used
    for e in range(used):
        tasks[e] = factory(env_node[e], e)
        calls.append((env_node[e], e))
        left[e] = tasks[e].steps
    rewards = [0.0] * n_nodes
    harvested = [False] * used

    def remaining(i):
        return sum(left[e] for e in range(used) if env_node[e] == i and left[e] > 0)

    def harvest():
        for e in range(used):
            if harvested[e] or left[e] > 0:
                continue
            harvested[e] = True
            rewards[env_node[e]] = max(rewards[env_node[e]], tasks[e].reward)
            if not leaf_parallel or not tasks[e].by_grasp:
                continue
            best, bw = -1, 0
            for i in range(n_nodes):
                w = remaining(i)
                if w > bw:
                    bw, best = w, i
            if best >= 0:
                env_node[e] = best
                tasks[e] = factory(best, e)
                calls.append((best, e))
                left[e] = tasks[e].steps
                harvested[e] = False

    harvest()
    rounds = 0
    while any(x > 0 for x in left):
        for e in range(used):
            if left[e] > 0:
                left[e] -= 1
        harvest()
        rounds += 1
    return np.array(rewards), calls, rounds


class ScriptedShard:
    """Host-side stand-in for a device shard (same begin/report/repurpose/step
    contract as DeviceShard), driven by a pure factory(node, env) -> Script.
    max_remaining == steps left (RolloutCursor::max_remaining == cap - pushes)."""

    def __init__(self, factory):
        self.factory = factory
        self.calls = []

    def begin(self, node_poses, node_meta, n_nodes, used, lo, hi, leaf_parallel, seed, iteration, cap):
        self.lo, self.hi, self.n_nodes = lo, hi, n_nodes
        base, rem = divmod(used, n_nodes)
        big = rem * (base + 1)
        self.node, self.left, self.task, self.harv = {}, {}, {}, {}
        for g in range(lo, hi):
            nd = g // (base + 1) if g < big else rem + (g - big) // base
            self._start(g, nd)

    def _start(self, g, nd):
        self.node[g] = nd
        self.task[g] = self.factory(nd, g)
        self.calls.append((nd, g))
        self.left[g] = self.task[g].steps
        self.harv[g] = False

    def report(self):
        W = np.zeros(self.n_nodes, np.int32)
        env, node, grasp, reward = [], [], [], []
        active = 0
        for g in range(self.lo, self.hi):
            if self.left[g] > 0:
                W[self.node[g]] += self.left[g]
                active += 1
            elif not self.harv[g]:
                self.harv[g] = True
                env.append(g)
                node.append(self.node[g])
                grasp.append(int(self.task[g].by_grasp))
                reward.append(self.task[g].reward)
        return (Records(np.array(env, np.int32), np.array(node, np.int32), np.array(grasp, np.uint8),
                        np.array(reward, np.float64)), W, active)

    def repurpose(self, env, node):
        for g, nd in zip(env, node):
            self._start(int(g), int(nd))

    def step(self):
        for g in range(self.lo, self.hi):
            if self.left[g] > 0:
                self.left[g] -= 1

    def counters(self):
        return np.zeros(4, np.int64)


def run_inprocess(n_nodes, n_envs, leaf_parallel, factory, shards=3):
    used = n_envs if leaf_parallel else n_nodes
    sh = [ScriptedShard(factory) for _ in range(shards)]
    ranges = [env_range(used, shards, r) for r in range(shards)]
    meta = np.zeros((n_nodes, 3), np.int32)
    rewards, ctr = sharded_simulate(sh, InProcessComm(), None, meta, n_envs, leaf_parallel, 0, 0, 10, ranges)
    return rewards, sorted(c for s in sh for c in s.calls), int(ctr[1])


# --- the reference's scripted lockstep cases (test_pmbs.cpp:255-320), as pure factories ---

def test_split_even_remainder_first():
    f = lambda node, env: Script(1, 0.01 * env, False)  # noqa: E731
    r, calls, _ = lockstep_reference(3, 8, True, f)
    assert calls == [(0, 0), (0, 1), (0, 2), (1, 3), (1, 4), (1, 5), (2, 6), (2, 7)]
    assert np.allclose(r, [0.02, 0.05, 0.07])
    rs, cs, _ = run_inprocess(3, 8, True, f)
    assert np.array_equal(rs, r) and cs == sorted(calls)


def test_no_leaf_parallel_one_env_per_node():
    f = lambda node, env: Script(0, 0.512, True)  # noqa: E731
    r, calls, _ = lockstep_reference(3, 8, False, f)
    assert calls == [(0, 0), (1, 1), (2, 2)] and np.all(r == 0.512)
    rs, cs, _ = run_inprocess(3, 8, False, f, shards=2)
    assert np.array_equal(rs, r) and cs == sorted(calls)


def test_repurpose_to_busiest_node():
    def f(node, env):
        if node == 0:
            return Script(0, 0.8, True)
        if node == 1:
            return Script(5, 0.3, True) if env == 1 else Script(3, 0.9, False)
        return Script(2, 0.5, False)
    r, calls, _ = lockstep_reference(3, 3, True, f)
    assert calls == [(0, 0), (1, 1), (2, 2), (1, 0)]
    assert np.allclose(r, [0.8, 0.9, 0.5])
    for shards in (1, 2, 3):
        rs, cs, _ = run_inprocess(3, 3, True, f, shards=shards)
        assert np.array_equal(rs, r) and cs == sorted(calls)


def test_max_aggregation():
    vals = [0.0, 0.512, 0.4096, 0.0]
    f = lambda node, env: Script(1, vals[env], False)  # noqa: E731
    r, _, _ = lockstep_reference(1, 4, True, f)
    assert r.tolist() == [0.512]
    assert run_inprocess(1, 4, True, f, shards=2)[0].tolist() == [0.512]


def _fuzz_factory(seed):
    def f(node, env):
        h = (node * 1000003 + env * 9176 + seed * 7919) % 1000
        return Script(h % 7, round(0.8 ** (h % 5), 6) if h % 3 else 0.0, h % 4 == 0)
    return f


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("shards", [2, 3, 5])
def test_fuzz_sharded_equals_reference(seed, shards):
    n_nodes, n_envs = 7 + seed, 40 + 3 * seed
    f = _fuzz_factory(seed)
    r, calls, rounds = lockstep_reference(n_nodes, n_envs, True, f)
    rs, cs, rr = run_inprocess(n_nodes, n_envs, True, f, shards=shards)
    assert np.array_equal(rs, r)
    assert cs == sorted(calls)
    assert rr == rounds


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, out_path, seed):
    import torch.distributed as dist

    from paper_2207_06649_b200.sharded import TorchComm
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    n_nodes, n_envs = 9, 57
    sh = ScriptedShard(_fuzz_factory(seed))
    rng = [env_range(n_envs, world, rank)]
    rewards, ctr = sharded_simulate([sh], TorchComm(), None, np.zeros((n_nodes, 3), np.int32), n_envs, True, 0, 0,
                                    10, rng)
    calls = np.array(sorted(sh.calls), np.int64).reshape(-1, 2)
    np.savez(f"{out_path}.{rank}.npz", rewards=rewards, calls=calls, rounds=ctr[1])
    dist.destroy_process_group()


@pytest.mark.parametrize("seed", [1, 4])
def test_gloo_two_ranks(tmp_path, seed):
    import torch.multiprocessing as mp
    port = _free_port()
    out = str(tmp_path / "res")
    mp.start_processes(_gloo_worker, args=(2, port, out, seed), nprocs=2, join=True, start_method="spawn")
    r, calls, rounds = lockstep_reference(9, 57, True, _fuzz_factory(seed))
    got_calls = []
    for rank in range(2):
        z = np.load(f"{out}.{rank}.npz")
        assert np.array_equal(z["rewards"], r)  # every rank holds the full reward vector
        assert int(z["rounds"]) == rounds
        got_calls += [tuple(c) for c in z["calls"].tolist()]
    assert sorted(got_calls) == sorted(calls)
