"""What-if model of an asynchronous lockstep from a PPG_STEP_TRACE record
file (latency-mode env-steps: env, round, start/end ns, done/by-grasp):
  lockstep makespan = sum over rounds of the slowest env-step of the round
  async makespan    = envs run their steps back to back; a step at round r
                      of an env that was re-purposed at the harvest of round
                      r-1 waits until every env finished round r-1
(unlimited parallelism: valid while active envs < resident warps).
python tools/async_model.py trace.bin
(the trace records need a library built with EXTRA_NVFLAGS=-DPPG_STEP_TRACE_BUILD)"""
import struct
import sys
from collections import defaultdict


def blocks(path):
    data = open(path, "rb").read()
    off = 0
    while off < len(data):
        marker, k = struct.unpack_from("<QQ", data, off)
        off += 16
        recs = [struct.unpack_from("<QQQQ", data, off + 32 * i) for i in range(k)]
        off += 32 * k
        yield recs


def model(recs):
    by_it = defaultdict(list)
    for r0, t0, t1, f in recs:
        env, rnd = r0 & 0xffffffff, r0 >> 32
        it = f >> 40
        by_it[it].append((env, rnd, (t1 - t0) * 1e-9, f & 1, (f >> 1) & 1))
    lock_total = async_total = chain_total = 0.0
    for it, steps in sorted(by_it.items()):
        rounds = defaultdict(float)
        per_env = defaultdict(list)
        for env, rnd, dt, done, byg in steps:
            rounds[rnd] = max(rounds[rnd], dt)
            per_env[env].append((rnd, dt, done, byg))
        lock = sum(rounds.values())
        rlist = sorted(rounds)
        # async: finish[r] = time every env finished its step of round r
        finish_round = {}
        env_t = defaultdict(float)
        env_steps = {e: sorted(v) for e, v in per_env.items()}
        ptr = {e: 0 for e in env_steps}
        prev_done = {}
        for r in rlist:
            end = 0.0
            for e, v in env_steps.items():
                i = ptr[e]
                if i >= len(v) or v[i][0] != r:
                    continue
                start = env_t[e]
                # re-purposed at harvest r-1 (its previous step ended done by grasp): wait for round r-1
                if e in prev_done and prev_done[e] == r - 1:
                    start = max(start, finish_round.get(r - 1, 0.0))
                t = start + v[i][1]
                env_t[e] = t
                if v[i][2] and v[i][3]:
                    prev_done[e] = r
                ptr[e] = i + 1
                end = max(end, t)
            finish_round[r] = max(end, finish_round.get(r - 1, 0.0))
        asy = max(env_t.values()) if env_t else 0.0
        # lower bound with no harvest waits at all (every re-purposing decided
        # the moment the env finishes): the longest env chain
        chain = max(sum(dt for _, dt, _, _ in v) for v in per_env.values()) if per_env else 0.0
        lock_total += lock
        async_total += asy
        chain_total += chain
    return lock_total, async_total, len(by_it), chain_total


if __name__ == "__main__":
    for i, recs in enumerate(blocks(sys.argv[1])):
        lk, asy, its, ch = model(recs)
        print(f"call {i}: {len(recs)} steps, {its} iterations: lockstep {lk * 1e3:.2f} ms, async {asy * 1e3:.2f} ms, "
              f"gain {lk / max(asy, 1e-12):.2f}x; no-wait chain bound {ch * 1e3:.2f} ms")
