"""The library-native multi-GPU path (csrc/multi.cu): the
rollout batch sharded by environment with ONE W all-reduce per lockstep
round and one reward max per iteration, the tree replicated.

Only one GPU exists here, so (as the profiling guide prescribes) wider worlds
are emulated without kernels that wait on each other: Context.multi(...,
emulate=True) puts G shards on one device and runs the exchange as one
kernel over every shard's buffer, ordered by events.  The shard kernels,
the harvest split and the host driver are the same code the NCCL transport
runs; NCCL itself runs with a world of 1 (ncclCommInitAll over one device,
and ncclCommInitRank as rank 0 of 1).  Everything is checked bit for bit
against the unmodified reference's goldens."""
import numpy as np
import pytest

import golden_io
from paper_2207_06649_b200 import Budget, Context, ParallelConfig, run_pmbs
from paper_2207_06649_b200.abi import default_params

pytestmark = pytest.mark.gpu


def _contexts():
    return [("emu2", lambda: Context.multi([0, 0], emulate=True)),
            ("emu3", lambda: Context.multi([0, 0, 0], emulate=True)),
            ("emu5", lambda: Context.multi([0] * 5, emulate=True)),
            ("nccl_all1", lambda: Context.multi([0])),
            ("nccl_rank1", lambda: Context.rank(0, 0, 1, None))]


@pytest.fixture(scope="module", params=[c[0] for c in _contexts()])
def mctx(request):
    c = dict(_contexts())[request.param]()
    yield request.param, c
    c.close()


def test_shard_info(mctx):
    name, c = mctx
    info = c.shard_info()
    world = {"emu2": 2, "emu3": 3, "emu5": 5}.get(name, 1)
    assert info["world"] == world and info["rank"] == 0
    assert info["transport"] == ("emulated" if name.startswith("emu") else "nccl")


def test_sharded_simulate_matches_reference_golden(mctx):
    """batch_simulate (pmbs.cpp:207-234) sharded: per-node rewards bitwise
    equal to the reference's, counters equal to the unsharded device run."""
    _, c = mctx
    cases = {cc["case_id"]: s for cc, s in golden_io.cases()}
    single = Context(0)
    try:
        for cid, ne, seed, cap, nposes, meta, rewards in golden_io.simulate_sets():
            for ctx in (c, single):
                ctx.set_params(default_params(n_envs=ne, rng_seed=seed))
                ctx.set_scene(cases[cid])
            r, ctr = c.simulate_arrays(nposes, meta, ne, True, seed, 0, cap)
            assert np.array_equal(r.view(np.uint64), rewards.view(np.uint64)), cid
            r1, ctr1 = single.simulate_arrays(nposes, meta, ne, True, seed, 0, cap)
            assert np.array_equal(ctr, ctr1), cid
            r, _ = c.simulate_arrays(nposes, meta, ne, False, seed, 0, cap)  # no leaf parallelism
            r1, _ = single.simulate_arrays(nposes, meta, ne, False, seed, 0, cap)
            assert np.array_equal(r.view(np.uint64), r1.view(np.uint64)), cid
    finally:
        single.close()


@pytest.mark.parametrize("idx", range(0, 20, 2))
def test_sharded_run_pmbs_first_decisions(mctx, idx):
    """run_pmbs on the sharded device tree == the reference fingerprint
    (action, tree signature, iterations, expansions, stop reason)."""
    _, c = mctx
    cc, st = golden_io.cases()[idx]
    d = cc["decision"]
    r = run_pmbs(st, ParallelConfig(rng_seed=int(cc["seed"])), ctx=c)
    assert list(r.action) == d["action"] and r.signature_fnv == int(d["sig_fnv"])
    assert (r.iterations, r.expansions, r.stop_reason) == (d["iterations"], d["expansions"], d["stop"])


def test_sharded_run_pmbs_wide(mctx):
    """Wide batches and C4 dense rings (the configurations C5 shards)."""
    from test_reference_pins_gpu import _wide_cfg, _wide_state
    _, c = mctx
    for rec in golden_io.wide():
        if rec["n_envs"] > 4096:
            continue
        r = run_pmbs(_wide_state(rec), _wide_cfg(rec), ctx=c)
        assert r.signature_fnv == int(rec["decision"]["sig_fnv"]), rec
        assert list(r.action) == rec["decision"]["action"]


def test_sharded_host_planner_and_seconds_budget():
    """The host-tree planner's batch_simulate routes through the sharded
    lockstep too; a seconds budget (each shard votes, max) terminates."""
    c = Context.multi([0, 0, 0], emulate=True)
    try:
        c.set_planner("host")
        for cc, st in golden_io.cases()[:6]:
            r = run_pmbs(st, ParallelConfig(rng_seed=int(cc["seed"])), ctx=c)
            assert r.signature_fnv == int(cc["decision"]["sig_fnv"])
        c.set_planner("device")
        cc, st = golden_io.cases()[17]
        r = run_pmbs(st, ParallelConfig(rng_seed=int(cc["seed"]), n_envs=256, budget=Budget.seconds(0.05)), ctx=c)
        assert r.iterations >= 1 and r.stop_reason in ("budget", "early_stop", "explored")
    finally:
        c.close()


def test_emulated_requires_one_device():
    from paper_2207_06649_b200 import DeviceError
    import paper_2207_06649_b200.abi as abi
    if abi.load_library().ppg_device_count() < 2:
        pytest.skip("needs two devices to build an invalid mixed-device emulation")
    with pytest.raises(DeviceError):
        Context.multi([0, 1], emulate=True)
