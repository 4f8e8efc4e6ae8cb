"""Device-resident PMBS tree (csrc/dtree.cu): one CUDA-graph
launch per PMBS iteration (selection with virtual visits, expansion +
attach, lockstep rollouts under a conditional WHILE node, backprop).  It must
reproduce the reference decision, tree signature and statistics exactly —
the same bar as the host tree (planner.cpp), which is run beside it."""
import numpy as np
import pytest

import golden_io
from paper_2207_06649_b200 import Budget, ParallelConfig, run_pmbs
from paper_2207_06649_b200.scenes import generate_case

pytestmark = pytest.mark.gpu


def _both(ctx, st, cfg):
    out = {}
    for mode in ("host", "device"):
        ctx.set_planner(mode)
        out[mode] = run_pmbs(st, cfg, ctx=ctx, want_signature=True)
    ctx.set_planner("auto")
    return out["host"], out["device"]


def _same(h, d):
    assert d.signature == h.signature
    assert list(d.action) == list(h.action)
    assert (d.iterations, d.expansions, d.stop_reason, d.final_tree_depth, d.n_nodes) == \
        (h.iterations, h.expansions, h.stop_reason, h.final_tree_depth, h.n_nodes)
    assert (d.env_steps, d.rollout_steps, d.lockstep_rounds) == (h.env_steps, h.rollout_steps, h.lockstep_rounds)


@pytest.mark.parametrize("idx", list(range(20)))
def test_device_tree_first_decisions(ctx, idx):
    """All 20 proj/cases first decisions (N_e = 64): device tree == host tree
    == the reference fingerprint."""
    c, st = golden_io.cases()[idx]
    d = c["decision"]
    h, dv = _both(ctx, st, ParallelConfig(rng_seed=int(c["seed"])))
    _same(h, dv)
    assert dv.signature_fnv == int(d["sig_fnv"]) and list(dv.action) == d["action"]


@pytest.mark.parametrize("n_envs,iters,leaf", [(1, 60, False), (7, 25, True), (300, 6, True), (300, 6, False),
                                               (5000, 3, True)])
def test_device_tree_budgets_and_widths(ctx, n_envs, iters, leaf):
    """Iteration budgets, narrow / wide batches (capacity growth, the lane-
    per-env kernels past the latency-mode limit) and no leaf parallelism."""
    c, st = golden_io.cases()[17]
    cfg = ParallelConfig(rng_seed=11, n_envs=n_envs, leaf_parallel=leaf, budget=Budget.iterations(iters))
    h, dv = _both(ctx, st, cfg)
    _same(h, dv)


@pytest.mark.parametrize("seed", [3, 8])
def test_device_tree_dense_deep(ctx, seed):
    """C4-like: dense ring motif (16 discs), deeper tree, wider action set."""
    st = generate_case(16, 0.0, seed, "ring")
    cfg = ParallelConfig(rng_seed=seed, n_envs=256, tree_depth=9, pushes_per_object=24,
                         budget=Budget.iterations(8))
    h, dv = _both(ctx, st, cfg)
    _same(h, dv)


def test_device_tree_acceptance_c1(ctx):
    """Reference acceptance C1 (N_e = 1, no leaf parallelism == serial MCTS)
    through the device tree, on the first 6 deep cases."""
    ctx.set_planner("device")
    try:
        for rec, st in golden_io.acceptance()["c1"][:6]:
            cfg = ParallelConfig(budget=Budget.iterations(500), rng_seed=rec["seed"], n_envs=1, leaf_parallel=False)
            r = run_pmbs(st, cfg, ctx=ctx)
            assert r.signature_fnv == int(rec["sig_fnv"]), rec["seed"]
            assert list(r.action) == rec["action"] and r.iterations == rec["iterations"]
    finally:
        ctx.set_planner("auto")


def test_device_tree_hybrid_rounds():
    """Large-batch lockstep rounds (warp sampler / graspable + lane physics)
    forced on (PPG_HYBRID_MIN=0) inside the device-tree graph: same trees."""
    from test_gpu_parity import _ctx_with
    c = _ctx_with(PPG_HYBRID_MIN=0)
    for idx in (12, 17):
        cc, st = golden_io.cases()[idx]
        d = cc["decision"]
        r = run_pmbs(st, ParallelConfig(rng_seed=int(cc["seed"])), ctx=c)
        assert list(r.action) == d["action"] and r.signature_fnv == int(d["sig_fnv"])
    _, st = golden_io.cases()[17]
    cfg = ParallelConfig(rng_seed=11, n_envs=300, budget=Budget.iterations(6))
    h, dv = _both(c, st, cfg)
    _same(h, dv)
    c.close()


@pytest.mark.parametrize("scene", ["case_18", "case_16", "ring18"])
def test_device_tree_adaptive_rounds(scene):
    """PPG_HYBRID_MIN=64: rounds with >= 64 active envs are hybrid, the rest
    one warp per env, switched per round on the device (disc scenes with the
    lane kernel); scenes without it (polygons: case_16, 18 discs) keep one
    fixed mode.  Must finish and equal the host tree."""
    from paper_2207_06649_b200.scenes import generate_case
    from test_gpu_parity import _ctx_with
    c = _ctx_with(PPG_HYBRID_MIN=64)
    if scene == "ring18":
        st = generate_case(18, 0.0, 5, "ring")
        cfg = ParallelConfig(rng_seed=5, n_envs=512, budget=Budget.iterations(3))
    else:
        cc, st = {x["case_id"]: (x, s) for x, s in golden_io.cases()}[scene]
        cfg = ParallelConfig(rng_seed=int(cc["seed"]), n_envs=512, budget=Budget.iterations(4))
    h, dv = _both(c, st, cfg)
    _same(h, dv)
    c.close()


@pytest.mark.parametrize("n,pf,depth,na", [(2, 0.0, 1, 16), (3, 1.0, 2, 32), (4, 0.5, 3, 8), (6, 0.0, 12, 16)])
def test_device_tree_small_scenes_and_shapes(ctx, n, pf, depth, na):
    """Tiny scenes (1-6 objects, discs / polygons), very shallow and deep
    trees, N_a from 8 to 32 (kMaxNa): device tree == host tree."""
    from paper_2207_06649_b200.scenes import generate_cases, _take
    from paper_2207_06649_b200.world import WorldState
    t, poses, ok = generate_cases(n, np.arange(500, 540), pf)
    found = errors = 0
    for k in np.nonzero(ok)[0]:
        st = WorldState(t.kind[k].copy(), t.radius[k].copy(), t.n_vertices[k].copy(), t.vertices[k].copy(),
                        poses[k].copy(), int(t.target_index[k]), 0.288, 0.0)
        cfg = ParallelConfig(rng_seed=int(k), n_envs=48, tree_depth=depth, pushes_per_object=na,
                             budget=Budget.iterations(6))
        try:
            h, dv = _both(ctx, st, cfg)
        except Exception as e:  # root graspable / no legal push: both trees must agree on the error
            ctx.set_planner("device")
            with pytest.raises(type(e)):
                run_pmbs(st, cfg, ctx=ctx)
            ctx.set_planner("auto")
            errors += 1
            continue
        _same(h, dv)
        found += 1
        if found == 3:
            break
    assert found + errors > 0
    assert found > 0 or n <= 3  # with 2-3 objects the target is often graspable at the root
