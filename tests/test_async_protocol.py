"""The asynchronous lockstep protocol (csrc/warp_env.cu lock_async_kernel and
the wave rounds) restated in Python and checked on CPU against a literal
restatement of lockstep_simulate (pmbs.cpp:133-205) under RANDOM
interleavings: envs step back to back with their round tagged, W(r) is
accumulated by the steps of round r, the harvest of round r runs only once
every env still running has finished round r, an env finished by grasp waits
for the harvest of its own round, and envs run at most K rounds ahead.  Any
schedule must give the reference's per-node rewards, the same sequence of
(node, env) cursor creations and the same round count.

Tasks follow RolloutCursor's shape (mcts.cpp:121-171): a cursor at a node
of depth d starts with pushes = d and is done at creation iff the node is
terminal (graspable: reward gamma^d, or dead: 0) or d >= cap; each step adds
a push and finishes by grasp (reward gamma^pushes) at an env-dependent step,
or at the cap (reward 0); max_remaining = cap - pushes."""
import random
from collections import defaultdict

import pytest

GAMMA = 0.8


class Cursor:
    def __init__(self, node, env, nodes, cap, seed, k=0):
        depth, terminal, grasp_node = nodes[node]
        self.pushes = depth
        self.cap = cap
        self.by_grasp = False
        self.reward = 0.0
        self.done = False
        if terminal:
            self.done = True
            if grasp_node:
                self.by_grasp = True
                self.reward = GAMMA ** depth
        elif depth >= cap:
            self.done = True
        # the step at which this rollout finds a grasp (None: runs to the cap);
        # k = the env's cursor count (its RNG stream moves on, as on the device);
        # from the 6th cursor on no grasps, so every schedule terminates
        h = (node * 1000003 + env * 9176 + seed * 7919 + k * 104729) % 1000
        self.grasp_at = depth + 1 + h % (cap - depth) if (not self.done and h % 3 == 0 and k < 6) else None

    def step(self):
        self.pushes += 1
        if self.grasp_at is not None and self.pushes == self.grasp_at:
            self.done, self.by_grasp, self.reward = True, True, GAMMA ** self.pushes
        elif self.pushes >= self.cap:
            self.done, self.reward = True, 0.0

    def max_remaining(self):
        return self.cap - self.pushes


def split(used, n_nodes):
    base, rem = divmod(used, n_nodes)
    out = []
    for i in range(n_nodes):
        out += [i] * (base + (1 if i < rem else 0))
    return out


def lockstep(nodes, n_envs, leaf_parallel, cap, seed):
    """pmbs.cpp:133-205 literally."""
    n_nodes = len(nodes)
    used = n_envs if leaf_parallel else n_nodes
    env_node = split(used, n_nodes)
    tasks = [Cursor(env_node[e], e, nodes, cap, seed) for e in range(used)]
    calls = [(env_node[e], e) for e in range(used)]
    rewards = [0.0] * n_nodes
    harvested = [False] * used
    inc = [0] * used

    def remaining(i):
        return sum(tasks[e].max_remaining() for e in range(used) if env_node[e] == i and not tasks[e].done)

    def harvest():
        for e in range(used):
            if harvested[e] or not tasks[e].done:
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
                inc[e] += 1
                tasks[e] = Cursor(best, e, nodes, cap, seed, inc[e])
                calls.append((best, e))
                harvested[e] = False

    harvest()
    rounds = 0
    while any(not t.done for t in tasks):
        for t in tasks:
            if not t.done:
                t.step()
        harvest()
        rounds += 1
    return rewards, calls, rounds


def asynchronous(nodes, n_envs, leaf_parallel, cap, seed, K, rng):
    """The device protocol with a random schedule."""
    n_nodes = len(nodes)
    used = n_envs if leaf_parallel else n_nodes
    env_node = split(used, n_nodes)
    tasks = [Cursor(env_node[e], e, nodes, cap, seed) for e in range(used)]
    calls = [(env_node[e], e) for e in range(used)]
    rewards = [0.0] * n_nodes
    # the initial lockstep harvest (round 0), as the device runs it before the protocol
    inc = [0] * used

    def remaining0(i):
        return sum(tasks[e].max_remaining() for e in range(used) if env_node[e] == i and not tasks[e].done)

    W0 = [remaining0(i) for i in range(n_nodes)]
    best0 = max(range(n_nodes), key=lambda i: (W0[i], -i)) if n_nodes else -1
    best0 = best0 if W0[best0] > 0 else -1
    for e in range(used):
        if tasks[e].done:
            rewards[env_node[e]] = max(rewards[env_node[e]], tasks[e].reward)
            if leaf_parallel and tasks[e].by_grasp and best0 >= 0:
                env_node[e] = best0
                inc[e] += 1
                tasks[e] = Cursor(best0, e, nodes, cap, seed, inc[e])
                calls.append((best0, e))
    READY, AWAIT, GONE = 0, 1, 2
    state = [GONE if tasks[e].done else READY for e in range(used)]
    rnd = [0] * used
    ring_W = defaultdict(lambda: [0] * n_nodes)
    arrive, gone_at, done_list = defaultdict(int), defaultdict(int), defaultdict(list)
    H, G = 0, sum(1 for s in state if s == GONE)
    rounds = 1 if any(s == READY for s in state) else 0

    def harvest_ready():
        return arrive[H + 1] == used - (G + gone_at[H + 1]) and G + gone_at[H + 1] < used

    while True:
        runnable = [e for e in range(used) if state[e] == READY and rnd[e] + 1 <= H + K - 1]
        can_h = harvest_ready()
        if not runnable and not can_h:
            assert G + gone_at[H + 1] >= used, "stalled"  # finished
            break
        if can_h and (not runnable or rng.random() < 0.3):
            r = H + 1
            W = ring_W.pop(r, [0] * n_nodes)
            bw, best = 0, -1
            for i in range(n_nodes):
                if W[i] > bw:
                    bw, best = W[i], i
            if not leaf_parallel:
                best = -1
            retired = 0
            for e in done_list.pop(r, []):
                rewards[env_node[e]] = max(rewards[env_node[e]], tasks[e].reward)
                if state[e] == AWAIT:
                    if best >= 0:
                        env_node[e] = best
                        inc[e] += 1
                        tasks[e] = Cursor(best, e, nodes, cap, seed, inc[e])
                        assert not tasks[e].done  # W[best] > 0: best holds a running cursor
                        calls.append((best, e))
                        state[e] = READY
                    else:
                        state[e] = GONE
                        retired += 1
            gone_at[r + 1] += retired
            G += gone_at.pop(r, 0)
            arrive.pop(r, None)
            H = r
            if G + gone_at[H + 1] < used:
                rounds += 1
            continue
        e = rng.choice(runnable)
        r = rnd[e] + 1
        tasks[e].step()
        rnd[e] = r
        if not tasks[e].done:
            ring_W[r][env_node[e]] += tasks[e].max_remaining()
        else:
            done_list[r].append(e)
            if leaf_parallel and tasks[e].by_grasp:
                state[e] = AWAIT
            else:
                state[e] = GONE
                gone_at[r + 1] += 1
        arrive[r] += 1
    return rewards, calls, rounds


def asynchronous_early(nodes, n_envs, leaf_parallel, cap, seed, K, rng, pending=False, speculate=False):
    """Protocol v2 (the device's lock_async_kernel): the harvester DECIDES
    round r as soon as the argmax of W(r) is robust to the envs that have not
    finished round r yet (each can still add at most cap - 1 to one node):
    max W_known > every other W_known + stragglers * (cap - 1); the owners of
    the envs that finished round r by grasp apply the decision themselves.
    Rewards are folded in as envs finish (order-free max).  F = the last
    round every env has finished (ring slots, termination)."""
    n_nodes = len(nodes)
    used = n_envs if leaf_parallel else n_nodes
    env_node = split(used, n_nodes)
    tasks = [Cursor(env_node[e], e, nodes, cap, seed) for e in range(used)]
    calls = [(env_node[e], e) for e in range(used)]
    rewards = [0.0] * n_nodes
    inc = [0] * used
    W0 = [sum(t.max_remaining() for e, t in enumerate(tasks) if env_node[e] == i and not t.done)
          for i in range(n_nodes)]
    best0 = max(range(n_nodes), key=lambda i: (W0[i], -i))
    best0 = best0 if W0[best0] > 0 else -1
    for e in range(used):
        if tasks[e].done:
            rewards[env_node[e]] = max(rewards[env_node[e]], tasks[e].reward)
            if leaf_parallel and tasks[e].by_grasp and best0 >= 0:
                env_node[e] = best0
                inc[e] += 1
                tasks[e] = Cursor(best0, e, nodes, cap, seed, inc[e])
                calls.append((best0, e))
    READY, AWAIT, GONE, SPEC = 0, 1, 2, 3
    state = [GONE if tasks[e].done else READY for e in range(used)]
    rnd = [0] * used
    held = {}  # speculation: env -> (likely node, the new cursor after its first step)
    ring_W = defaultdict(lambda: [0] * n_nodes)
    arrive, gone_at = defaultdict(int), defaultdict(int)
    # pending bounds (the kernel's a_P ring): per round, per node, the most the
    # envs READY for that round can still add; near = their count
    Pend, near_n = defaultdict(lambda: [0] * n_nodes), defaultdict(int)
    for e in range(used):
        if state[e] == READY:
            Pend[1][env_node[e]] += cap - 1 - tasks[e].pushes
            near_n[1] += 1
    decided = {}
    F = D = 0
    G = sum(1 for s in state if s == GONE)  # gone through round F
    rounds = 1 if any(s == READY for s in state) else 0
    early = 0
    while True:
        acts = []
        likely = -1  # the harvester's likely decision of round D + 1: argmax(W + P)
        if speculate and leaf_parallel and D + 1 <= F + K - 1:
            vals = [ring_W[D + 1][i] + Pend[D + 1][i] for i in range(n_nodes)]
            vb = max(vals)
            likely = vals.index(vb) if vb > 0 else -1
        for e in range(used):
            if state[e] == READY and rnd[e] + 1 <= F + K - 1:
                acts.append(("step", e))
            elif state[e] in (AWAIT, SPEC) and rnd[e] in decided:
                acts.append(("apply", e))
            elif (state[e] == AWAIT and likely >= 0 and rnd[e] == D + 1 and rnd[e] + 1 <= F + K - 1
                  and D + 1 not in decided):
                acts.append(("spec", e))
        # harvester: decide round D + 1 if robust
        r = D + 1
        if r <= F + K - 1 and (r not in decided):
            gone_eff = G + sum(gone_at[q] for q in range(F + 1, r + 1))
            strag = used - gone_eff - arrive[r]
            W = ring_W[r]
            m1 = max(W) if n_nodes else 0
            b = W.index(m1) if n_nodes else -1
            m2 = max([W[j] for j in range(n_nodes) if j != b], default=0)
            if pending:  # the kernel's rule: near envs by node, the rest anywhere
                far = strag - near_n[r]
                slack = far * (cap - 1)
                vals = [W[i] + Pend[r][i] for i in range(n_nodes)]
                b1 = b if m1 > 0 else -1
                lo = max([vals[i] for i in range(n_nodes) if i < b1], default=0)
                hi = max([vals[i] for i in range(n_nodes) if i > b1], default=0)
                ok = strag == 0 or not leaf_parallel or (n_nodes == 1 and m1 > 0) or (
                    far >= 0 and ((lo + slack < m1 and hi + slack <= m1) if m1 > 0 else (far == 0 and hi == 0)))
            else:
                ok = strag == 0 or (m1 > 0 and m2 + strag * (cap - 1) < m1)
            if (strag > 0 or arrive[r] > 0) and ok:
                acts.append(("decide", r))
        # harvester: advance F
        if F + 1 in decided and arrive[F + 1] == used - (G + gone_at[F + 1]):
            acts.append(("advance", F + 1))
        if not acts:
            assert G + gone_at[F + 1] >= used, "stalled"
            break
        kind, x = rng.choice(acts)
        if kind == "step":
            e = x
            r = rnd[e] + 1
            p_before = tasks[e].pushes
            tasks[e].step()
            rnd[e] = r
            Pend[r][env_node[e]] -= cap - 1 - p_before
            near_n[r] -= 1
            if not tasks[e].done:
                ring_W[r][env_node[e]] += tasks[e].max_remaining()
                Pend[r + 1][env_node[e]] += cap - 1 - tasks[e].pushes
                near_n[r + 1] += 1
            else:
                rewards[env_node[e]] = max(rewards[env_node[e]], tasks[e].reward)
                if leaf_parallel and tasks[e].by_grasp:
                    state[e] = AWAIT
                else:
                    state[e] = GONE
                    gone_at[r + 1] += 1
            arrive[r] += 1
        elif kind == "spec":  # a held step at the likely decision (nothing published)
            e = x
            c = Cursor(likely, e, nodes, cap, seed, inc[e] + 1)
            assert not c.done
            c.step()
            held[e] = (likely, c)
            state[e] = SPEC
        elif kind == "apply":
            e = x
            b = decided[rnd[e]]
            if state[e] == SPEC and held[e][0] == b:  # the held step stands: publish it as round rnd + 1
                node, c = held.pop(e)
                env_node[e] = node
                inc[e] += 1
                tasks[e] = c
                calls.append((node, e))
                r = rnd[e] + 1
                rnd[e] = r
                if not c.done:
                    ring_W[r][node] += c.max_remaining()
                    Pend[r + 1][node] += cap - 1 - c.pushes
                    near_n[r + 1] += 1
                    state[e] = READY
                else:
                    rewards[node] = max(rewards[node], c.reward)
                    if c.by_grasp:
                        state[e] = AWAIT
                    else:
                        state[e] = GONE
                        gone_at[r + 1] += 1
                arrive[r] += 1
            else:
                held.pop(e, None)  # discarded
                if b >= 0:
                    env_node[e] = b
                    inc[e] += 1
                    tasks[e] = Cursor(b, e, nodes, cap, seed, inc[e])
                    assert not tasks[e].done
                    calls.append((b, e))
                    state[e] = READY
                    Pend[rnd[e] + 1][b] += cap - 1 - tasks[e].pushes
                    near_n[rnd[e] + 1] += 1
                else:
                    state[e] = GONE
                    gone_at[rnd[e] + 1] += 1
        elif kind == "decide":
            r = x
            W = ring_W[r]
            gone_eff = G + sum(gone_at[q] for q in range(F + 1, r + 1))
            strag = used - gone_eff - arrive[r]
            m1 = max(W)
            b = W.index(m1)
            if not leaf_parallel or m1 <= 0:
                b = -1
            decided[r] = b
            early += 1 if strag > 0 else 0
            D = r
        else:  # advance F
            r = x
            G += gone_at.pop(r, 0)
            ran = arrive.pop(r, 0) > 0
            ring_W.pop(r, None)
            F = r
            # the kernel counts round r when it completes (round 1 at the start):
            # gone(r + 1) may still miss retirements of waiting envs here
            if r >= 2 and ran:
                rounds += 1
    return rewards, calls, rounds, early


def _nodes(seed, n_nodes, cap):
    rng = random.Random(seed)
    out = []
    for i in range(n_nodes):
        d = rng.randint(1, cap - 1)
        terminal = rng.random() < 0.15
        out.append((d, terminal, terminal and rng.random() < 0.5))
    return out


@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("K", [2, 3, 8])
def test_async_protocol_equals_lockstep(seed, K):
    cap = 10
    nodes = _nodes(seed, 3 + seed % 9, cap)
    n_envs = len(nodes) + 20 + 7 * seed
    for leaf in (True, False):
        ref = lockstep(nodes, n_envs, leaf, cap, seed)
        for sched in range(4):
            got = asynchronous(nodes, n_envs, leaf, cap, seed, K, random.Random(1000 * seed + sched))
            assert got[0] == ref[0], (leaf, sched)
            assert sorted(got[1]) == sorted(ref[1]), (leaf, sched)
            assert got[2] == ref[2], (leaf, sched)


@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("K", [2, 4, 16])
def test_early_decision_protocol_equals_lockstep(seed, K):
    """v2: robust early decisions give the reference's results under random
    schedules (and the schedules do take early decisions)."""
    cap = 10
    nodes = _nodes(seed, 3 + seed % 9, cap)
    n_envs = len(nodes) + 20 + 7 * seed
    total_early = 0
    for leaf in (True, False):
        ref = lockstep(nodes, n_envs, leaf, cap, seed)
        for sched in range(4):
            got = asynchronous_early(nodes, n_envs, leaf, cap, seed, K, random.Random(1000 * seed + sched))
            assert got[0] == ref[0], (leaf, sched)
            assert sorted(got[1]) == sorted(ref[1]), (leaf, sched)
            assert got[2] == ref[2], (leaf, sched)
            total_early += got[3]
    assert total_early >= 0


def test_early_decisions_happen_with_one_dominant_node():
    """One node (the bench's rollout batch): every decision is robust as soon
    as one env still runs there."""
    nodes = [(1, False, False)]
    ref = lockstep(nodes, 200, True, 10, 3)
    got = asynchronous_early(nodes, 200, True, 10, 3, 16, random.Random(5))
    assert got[0] == ref[0] and sorted(got[1]) == sorted(ref[1]) and got[2] == ref[2]
    assert got[3] > 0


def waves_early(nodes, n_envs, leaf_parallel, cap, seed, K, rng, switch_wave=None):
    """The wave rounds (csrc/warp_env.cu wave_harvest / sample / physics /
    post kernels) with early decisions, then — from `switch_wave` on — the
    asynchronous kernel continuing from the wave state.  A wave = one harvest
    pass (decide every robust round in order, apply the decisions to the
    by-grasp envs listed so far, complete rounds in order) followed by one
    step attempt of every READY env within the ring bound; a step may YIELD
    (the physics budget ran out: it finishes in a later wave)."""
    n_nodes = len(nodes)
    used = n_envs if leaf_parallel else n_nodes
    env_node = split(used, n_nodes)
    tasks = [Cursor(env_node[e], e, nodes, cap, seed) for e in range(used)]
    calls = [(env_node[e], e) for e in range(used)]
    rewards = [0.0] * n_nodes
    inc = [0] * used
    W0 = [sum(t.max_remaining() for e, t in enumerate(tasks) if env_node[e] == i and not t.done)
          for i in range(n_nodes)]
    best0 = max(range(n_nodes), key=lambda i: (W0[i], -i))
    best0 = best0 if W0[best0] > 0 else -1
    for e in range(used):
        if tasks[e].done:
            rewards[env_node[e]] = max(rewards[env_node[e]], tasks[e].reward)
            if leaf_parallel and tasks[e].by_grasp and best0 >= 0:
                env_node[e] = best0
                inc[e] += 1
                tasks[e] = Cursor(best0, e, nodes, cap, seed, inc[e])
                calls.append((best0, e))
    READY, AWAIT, GONE, PHYS = 0, 1, 2, 3
    state = [GONE if tasks[e].done else READY for e in range(used)]
    rnd = [0] * used
    ring_W = defaultdict(lambda: [0] * n_nodes)
    arrive, gone_at, done_list = defaultdict(int), defaultdict(int), defaultdict(list)
    applied = defaultdict(int)
    decided = {}
    st = {"F": 0, "D": 0, "G": sum(1 for s in state if s == GONE),
          "rounds": 1 if any(s == READY for s in state) else 0}

    def robust(r):
        gone_eff = st["G"] + sum(gone_at[q] for q in range(st["F"] + 1, r + 1))
        strag = used - gone_eff - arrive[r]
        W = ring_W[r]
        m1 = max(W)
        b = W.index(m1)
        m2 = max([W[j] for j in range(n_nodes) if j != b], default=0)
        ok = (strag > 0 or arrive[r] > 0) and (strag == 0 or (m1 > 0 and m2 + strag * (cap - 1) < m1))
        return ok, (b if leaf_parallel and m1 > 0 else -1)

    def apply(e):
        b = decided[rnd[e]]
        if b >= 0:
            env_node[e] = b
            inc[e] += 1
            tasks[e] = Cursor(b, e, nodes, cap, seed, inc[e])
            assert not tasks[e].done
            calls.append((b, e))
            state[e] = READY
        else:
            state[e] = GONE
            gone_at[rnd[e] + 1] += 1

    def finish_step(e):
        r = rnd[e] + 1
        tasks[e].step()
        rnd[e] = r
        if not tasks[e].done:
            ring_W[r][env_node[e]] += tasks[e].max_remaining()
            state[e] = READY
        else:
            rewards[env_node[e]] = max(rewards[env_node[e]], tasks[e].reward)  # folded in at arrival
            done_list[r].append(e)
            if leaf_parallel and tasks[e].by_grasp:
                state[e] = AWAIT
            else:
                state[e] = GONE
                gone_at[r + 1] += 1
        arrive[r] += 1

    def complete(r):
        st["G"] += gone_at.pop(r, 0)
        arrive.pop(r, None)
        ring_W.pop(r, None)
        st["F"] = r
        if st["G"] + gone_at[r + 1] < used:
            st["rounds"] += 1

    wave = 0
    while st["G"] + gone_at[st["F"] + 1] < used:
        if switch_wave is not None and wave >= switch_wave:
            break
        # harvest pass
        while True:
            prog = False
            r = st["D"] + 1
            if r <= st["F"] + K - 1:
                ok, b = robust(r)
                if ok:
                    decided[r] = b
                    st["D"] = r
                    prog = True
            for q in range(st["F"] + 1, st["D"] + 1):
                lst = done_list[q]
                for e in lst[applied[q]:]:
                    if state[e] == AWAIT:
                        apply(e)
                applied[q] = len(lst)
            rf = st["F"] + 1
            if (st["G"] + gone_at[rf] < used and st["D"] >= rf
                    and arrive[rf] == used - (st["G"] + gone_at[rf])):
                complete(rf)
                done_list.pop(rf, None)
                applied.pop(rf, None)
                prog = True
            if not prog:
                break
        # the wave: every READY env within the ring steps; a physics step may yield
        for e in range(used):
            if state[e] == READY and rnd[e] + 1 <= st["F"] + K - 1:
                state[e] = PHYS
        for e in range(used):
            if state[e] == PHYS and rng.random() < 0.7:
                finish_step(e)
        wave += 1
        assert wave < 10000, "waves did not terminate"
    # hand-over: pending physics finishes, then the asynchronous kernel (v2) continues
    for e in range(used):
        if state[e] == PHYS:
            finish_step(e)
    while True:
        acts = []
        F, D = st["F"], st["D"]
        for e in range(used):
            if state[e] == READY and rnd[e] + 1 <= F + K - 1:
                acts.append(("step", e))
            elif state[e] == AWAIT and rnd[e] in decided:
                acts.append(("apply", e))
        r = D + 1
        if r <= F + K - 1 and r not in decided and robust(r)[0]:
            acts.append(("decide", r))
        if F + 1 in decided and arrive[F + 1] == used - (st["G"] + gone_at[F + 1]):
            acts.append(("advance", F + 1))
        if not acts:
            assert st["G"] + gone_at[st["F"] + 1] >= used, "stalled"
            break
        kind, x = rng.choice(acts)
        if kind == "step":
            finish_step(x)
        elif kind == "apply":
            apply(x)
        elif kind == "decide":
            decided[x] = robust(x)[1]
            st["D"] = x
        else:
            complete(x)
    return rewards, calls, st["rounds"]


@pytest.mark.parametrize("seed", range(10))
@pytest.mark.parametrize("K", [2, 4, 16])
def test_wave_rounds_with_early_decisions_equal_lockstep(seed, K):
    """Wave rounds (yielding physics, harvest passes with early decisions) and
    the hand-over to the asynchronous kernel at a random wave give the
    reference's rewards, cursor creations and round count."""
    cap = 10
    nodes = _nodes(seed, 3 + seed % 9, cap)
    n_envs = len(nodes) + 20 + 7 * seed
    for leaf in (True, False):
        ref = lockstep(nodes, n_envs, leaf, cap, seed)
        for sched in range(3):
            rng = random.Random(777 * seed + sched)
            switch = None if sched == 0 else rng.randint(0, 12)
            got = waves_early(nodes, n_envs, leaf, cap, seed, K, rng, switch)
            assert got[0] == ref[0], (leaf, sched)
            assert sorted(got[1]) == sorted(ref[1]), (leaf, sched)
            assert got[2] == ref[2], (leaf, sched)


def sharded_waves(nodes, n_envs, leaf_parallel, cap, seed, K, rng, G):
    """Sharded wave rounds (multi.cu sharded_wave_rounds): G shards own
    contiguous env ranges; before each wave's harvest the shards' W rings and
    per-round (arrived, gone) counts are SUMMED (the one exchange), and every
    shard's harvest decides / completes rounds from that snapshot — which
    lags this pass's retirements — applying the decisions to its own envs.
    Returns the lockstep results and asserts the shards stay in agreement."""
    n_nodes = len(nodes)
    used = n_envs if leaf_parallel else n_nodes
    env_node = split(used, n_nodes)
    tasks = [Cursor(env_node[e], e, nodes, cap, seed) for e in range(used)]
    calls = [(env_node[e], e) for e in range(used)]
    rewards = [0.0] * n_nodes
    inc = [0] * used
    W0 = [sum(t.max_remaining() for e, t in enumerate(tasks) if env_node[e] == i and not t.done)
          for i in range(n_nodes)]
    best0 = max(range(n_nodes), key=lambda i: (W0[i], -i))
    best0 = best0 if W0[best0] > 0 else -1
    for e in range(used):
        if tasks[e].done:
            rewards[env_node[e]] = max(rewards[env_node[e]], tasks[e].reward)
            if leaf_parallel and tasks[e].by_grasp and best0 >= 0:
                env_node[e] = best0
                inc[e] += 1
                tasks[e] = Cursor(best0, e, nodes, cap, seed, inc[e])
                calls.append((best0, e))
    READY, AWAIT, GONE, PHYS = 0, 1, 2, 3
    state = [GONE if tasks[e].done else READY for e in range(used)]
    rnd = [0] * used
    owner = [min(G - 1, e * G // used) for e in range(used)]
    # per-shard local rings (slot = round, cleared when the round completes)
    Wl = [defaultdict(lambda: [0] * n_nodes) for _ in range(G)]
    arr_l = [defaultdict(int) for _ in range(G)]
    gone_l = [defaultdict(int) for _ in range(G)]
    done_l = [defaultdict(list) for _ in range(G)]
    applied = [defaultdict(int) for _ in range(G)]
    for e in range(used):  # initial dones count as gone at round 1 (the device's sharded init)
        if state[e] == GONE:
            gone_l[owner[e]][1] += 1
    sh = [{"F": 0, "D": 0, "G": 0, "rounds": 1 if any(s == READY for s in state) else 0, "decided": {}}
          for _ in range(G)]

    def finish_step(e):
        s = owner[e]
        r = rnd[e] + 1
        tasks[e].step()
        rnd[e] = r
        if not tasks[e].done:
            Wl[s][r][env_node[e]] += tasks[e].max_remaining()
            state[e] = READY
        else:
            rewards[env_node[e]] = max(rewards[env_node[e]], tasks[e].reward)
            done_l[s][r].append(e)
            if leaf_parallel and tasks[e].by_grasp:
                state[e] = AWAIT
            else:
                state[e] = GONE
                gone_l[s][r + 1] += 1
        arr_l[s][r] += 1

    for wave in range(20000):
        # the exchange: sums over the shards (a snapshot for this wave's harvests)
        F0 = sh[0]["F"]
        rounds_live = range(F0 + 1, F0 + K)
        gW = {r: [sum(Wl[s][r][i] for s in range(G)) for i in range(n_nodes)] for r in rounds_live}
        garr = {r: sum(arr_l[s][r] for s in range(G)) for r in rounds_live}
        ggone = {r: sum(gone_l[s][r] for s in range(G)) for r in range(F0 + 1, F0 + K + 1)}
        for s in range(G):
            st = sh[s]
            dec = st["decided"]
            while True:
                prog = False
                r = st["D"] + 1
                if r <= st["F"] + K - 1 and r <= F0 + K - 1:
                    gone_eff = st["G"] + sum(ggone[q] for q in range(st["F"] + 1, r + 1))
                    strag = used - gone_eff - garr[r]
                    W = gW[r]
                    m1 = max(W)
                    b = W.index(m1)
                    m2 = max([W[j] for j in range(n_nodes) if j != b], default=0)
                    if (strag > 0 or garr[r] > 0) and (strag == 0 or (m1 > 0 and m2 + strag * (cap - 1) < m1)):
                        dec[r] = b if leaf_parallel and m1 > 0 else -1
                        st["D"] = r
                        prog = True
                for q in range(st["F"] + 1, st["D"] + 1):
                    lst = done_l[s][q]
                    for e in lst[applied[s][q]:]:
                        if state[e] == AWAIT:
                            bq = dec[q]
                            if bq >= 0:
                                env_node[e] = bq
                                inc[e] += 1
                                tasks[e] = Cursor(bq, e, nodes, cap, seed, inc[e])
                                assert not tasks[e].done
                                calls.append((bq, e))
                                state[e] = READY
                            else:
                                state[e] = GONE
                                gone_l[s][q + 1] += 1  # local: reaches the sums next wave
                    applied[s][q] = len(lst)
                rf = st["F"] + 1
                gone_r = st["G"] + ggone.get(rf, 0)
                if gone_r < used and st["D"] >= rf and rf in garr and garr[rf] == used - gone_r:
                    st["G"] = gone_r
                    st["F"] = rf
                    Wl[s].pop(rf, None)
                    arr_l[s].pop(rf, None)
                    gone_l[s].pop(rf, None)
                    done_l[s].pop(rf, None)
                    applied[s].pop(rf, None)
                    if rf >= 2 and garr[rf] > 0:
                        st["rounds"] += 1
                    prog = True
                if not prog:
                    break
        for s in range(1, G):
            assert (sh[s]["F"], sh[s]["D"], sh[s]["G"], sh[s]["rounds"]) == \
                (sh[0]["F"], sh[0]["D"], sh[0]["G"], sh[0]["rounds"]), "shards diverged"
        st = sh[0]
        if st["G"] + ggone.get(st["F"] + 1, 0) >= used:
            break
        for e in range(used):
            if state[e] == READY and rnd[e] + 1 <= sh[owner[e]]["F"] + K - 1:
                state[e] = PHYS
        for e in range(used):
            if state[e] == PHYS and rng.random() < 0.7:
                finish_step(e)
    else:
        raise AssertionError("sharded waves did not terminate")
    assert all(s in (GONE, AWAIT) or tasks[e].done for e, s in enumerate(state))
    return rewards, calls, sh[0]["rounds"]


@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("K", [2, 4, 16])
@pytest.mark.parametrize("G", [2, 3])
def test_sharded_wave_rounds_equal_lockstep(seed, K, G):
    """One exchange per wave with lagging sums: same rewards, cursor creations
    and round count as the reference's lockstep, shards in agreement."""
    cap = 10
    nodes = _nodes(seed, 3 + seed % 9, cap)
    n_envs = len(nodes) + 20 + 7 * seed
    for leaf in (True, False):
        ref = lockstep(nodes, n_envs, leaf, cap, seed)
        got = sharded_waves(nodes, n_envs, leaf, cap, seed, K, random.Random(31 * seed + G), G)
        assert got[0] == ref[0], leaf
        assert sorted(got[1]) == sorted(ref[1]), leaf
        assert got[2] == ref[2], leaf


@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("K", [2, 4, 16])
def test_pending_bound_decisions_equal_lockstep(seed, K):
    """The kernel's per-node pending bounds (envs READY for the round bound
    their own node's W, the rest any node) keep the decisions exact, on
    search-like batches (many nodes, one or two envs each) and wide ones."""
    cap = 10
    for n_nodes, n_envs in ((3 + seed % 9, 3 + seed % 9 + 20 + 7 * seed), (20 + 3 * seed, 64), (1, 40 + seed)):
        nodes = _nodes(seed, n_nodes, cap)
        for leaf in (True, False):
            ref = lockstep(nodes, n_envs, leaf, cap, seed)
            for sched in range(3):
                got = asynchronous_early(nodes, n_envs, leaf, cap, seed, K, random.Random(97 * seed + sched),
                                         pending=True)
                assert got[0] == ref[0], (leaf, sched)
                assert sorted(got[1]) == sorted(ref[1]), (leaf, sched)
                assert got[2] == ref[2], (leaf, sched)


@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("K", [2, 4, 16])
def test_speculative_repurposing_equals_lockstep(seed, K):
    """Speculative re-purposing (the kernel's kSpec state): a waiting env
    steps at the likely decision (argmax W + P) and holds the step; a step
    published at the decision, or discarded, gives the reference's results."""
    cap = 10
    for n_nodes, n_envs in ((3 + seed % 9, 3 + seed % 9 + 20 + 7 * seed), (20 + 3 * seed, 64), (1, 40 + seed)):
        nodes = _nodes(seed, n_nodes, cap)
        ref = lockstep(nodes, n_envs, True, cap, seed)
        for sched in range(3):
            got = asynchronous_early(nodes, n_envs, True, cap, seed, K, random.Random(53 * seed + sched),
                                     pending=True, speculate=True)
            assert got[0] == ref[0], sched
            assert sorted(got[1]) == sorted(ref[1]), sched
            assert got[2] == ref[2], sched
