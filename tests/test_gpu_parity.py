"""GPU parity: the CUDA path through the C-ABI against the golden fixtures
(made by the unmodified reference) and the CPU oracle.  Everything is
bit-exact — disc and polygon scenes (the device sincos is a port of the
reference's glibc __sincos_fma)."""
import numpy as np
import pytest

import golden_io
from oracle import port
from paper_2207_06649_b200 import ParallelConfig, SearchError, ShapeTable, default_params
from paper_2207_06649_b200 import batch_resolve, graspable, run_pmbs, sample_pushes
from paper_2207_06649_b200.api import Budget, GripperTip, SimParams, SimError, resolve_push

pytestmark = pytest.mark.gpu
P = default_params()


def _bitwise(a, b):
    return np.all(a.view(np.uint64) == b.view(np.uint64), axis=tuple(range(1, a.ndim)))


@pytest.mark.parametrize("name", ["discs", "ring16", "hard18"])
def test_batch_resolve_discs_bitwise(ctx, name):
    t, poses, pushes, status, digests, out_ref = golden_io.resolve_set(name)
    ctx.set_params(P)
    out, st, resid = ctx.batch_resolve_arrays(t, poses, pushes)
    assert np.array_equal(st, status)
    ok = status == 0
    assert _bitwise(out[ok], out_ref[ok]).all()
    assert np.array_equal(port.state_digests(t, out)[ok], digests[ok])
    assert np.all(out[~ok] == 0.0)
    assert np.all(resid[status == 2] > P.eps_pen)


def test_batch_resolve_polygons(ctx):
    """Polygon scenes (generate_case ShapeMix{0.35}): bitwise, through the
    device port of glibc's sincos."""
    t, poses, pushes, status, digests, out_ref = golden_io.resolve_set("polygons")
    ctx.set_params(P)
    out, st, _ = ctx.batch_resolve_arrays(t, poses, pushes)
    assert np.array_equal(st, status)
    assert _bitwise(out, out_ref).all()
    assert np.array_equal(port.state_digests(t, out), digests)


def test_batch_resolve_shared_scene_and_reference_api(ctx):
    cases = golden_io.cases()
    c, st = cases[12]
    sp = port.sample_pushes(st, P)
    res = batch_resolve([st] * len(sp), list(sp), GripperTip(), SimParams(), ctx=ctx)
    exp, est, _ = port.batch_resolve(ShapeTable.shared(st), np.repeat(st.poses[None], len(sp), 0), sp, P)
    for k, r in enumerate(res):
        assert r.ok() == (est[k] == 0)
        if r.ok():
            assert _bitwise(r.state.poses[None], exp[k][None]).all()


def test_batch_resolve_edge_cases(ctx):
    c, st = golden_io.cases()[0]
    # empty batch
    assert batch_resolve([], [], ctx=ctx) == []
    # size mismatch -> SimError (push_sim.cpp:136-137)
    with pytest.raises(SimError):
        batch_resolve([st], [], ctx=ctx)
    # start collision -> per-element error, siblings unaffected (test_pushworld.cpp:321-330)
    good = port.sample_pushes(st, P)[0]
    tgt = st.poses[0]
    bad = np.array([tgt[0], tgt[1], tgt[0] + 0.05, tgt[1]])
    res = batch_resolve([st, st], [bad, good], ctx=ctx)
    assert not res[0].ok() and "collides" in res[0].error
    assert res[1].ok()
    with pytest.raises(SimError):
        resolve_push(st, bad, ctx=ctx)


def test_single_disc_closed_form(ctx):
    """test_pushworld.cpp:170-182: x = 0.05 - gap within 1e-12 relative."""
    from paper_2207_06649_b200.world import WorldState
    r = 0.016
    st = WorldState.from_objects([{"kind": "disc", "radius": r, "pose": [0.0, 0.0, 0.0]}])
    gap = 0.004
    sx = -(r + 0.012 + gap)
    out = resolve_push(st, [sx, 0.0, sx + 0.05, 0.0], ctx=ctx)
    assert abs(out.poses[0, 0] - (0.05 - gap)) <= 1e-12 * (0.05 - gap)
    assert out.poses[0, 1] == 0.0 and out.poses[0, 2] == 0.0


def test_sample_and_grasp_cases(ctx):
    ctx.set_params(P)
    for c, st in golden_io.cases():
        sp = sample_pushes(st, 16, ctx=ctx)
        assert len(sp) == c["n_pushes"], c["case_id"]
        assert golden_io.fnv_bytes(sp.tobytes()) == int(c["pushes_fnv"]), c["case_id"]
        g = graspable(st, ctx=ctx)
        assert g.graspable == c["graspable"], c["case_id"]
        assert g.margin == c["margin"]
        assert (list(g.best) if g.best else [0.0, 0.0, -1]) == c["best"]


def test_expand_matches_oracle(ctx):
    ctx.set_params(P)
    for c, st in golden_io.cases()[10:14]:
        ctx.set_scene(st)
        sp = port.sample_pushes(st, P)
        parents = np.repeat(st.poses[None], len(sp), 0)
        child, status, g, nu, un = ctx.expand_arrays(parents, sp)
        exp, est, _ = port.batch_resolve(ShapeTable.shared(st), parents, sp, P)
        assert np.array_equal(status, est)
        for k in range(len(sp)):
            if est[k] != 0:
                assert _bitwise(child[k][None], parents[k][None]).all() and nu[k] == 0
                continue
            assert _bitwise(child[k][None], exp[k][None]).all()
            s2 = st.with_poses(exp[k])
            sp2 = port.sample_pushes(s2, P)
            assert nu[k] == len(sp2)
            assert _bitwise(un[k, :nu[k]][None], sp2[None]).all()
            assert bool(g[k]) == port.graspable(s2, P)[0]


def test_simulate_matches_reference_golden(ctx):
    cases = {c["case_id"]: st for c, st in golden_io.cases()}
    for cid, ne, seed, cap, poses, meta, rewards in golden_io.simulate_sets():
        st = cases[cid]
        ctx.set_params(default_params(n_envs=ne, rng_seed=seed))
        ctx.set_scene(st)
        r, ctr = ctx.simulate_arrays(poses, meta, ne, True, seed, 0, cap)
        assert np.array_equal(r, rewards), cid
        ro, co = port.simulate(st, poses, meta, ne, True, seed, 0, cap, default_params(n_envs=ne))
        assert np.array_equal(ctr, co), cid


def test_simulate_no_leaf_parallel_and_validation(ctx):
    c, st = golden_io.cases()[12]
    ctx.set_params(P)
    ctx.set_scene(st)
    sp = port.sample_pushes(st, P)[:5]
    exp, est, _ = port.batch_resolve(ShapeTable.shared(st), np.repeat(st.poses[None], 5, 0), sp, P)
    meta = np.array([[1, 0, 0]] * 5, np.int32)
    r, _ = ctx.simulate_arrays(exp, meta, 8, False, 3, 1, 10)
    ro, _ = port.simulate(st, exp, meta, 8, False, 3, 1, 10, P)
    assert np.array_equal(r, ro)
    with pytest.raises(ValueError):
        ctx.simulate_arrays(exp, meta, 4, True, 3, 1, 10)


@pytest.mark.parametrize("idx", list(range(20)))
def test_first_decision_fingerprints(ctx, idx):
    """SURVEY A.5 / tests/golden/cases.json: run_pmbs at the reference
    defaults (N_e = 64) reproduces the reference's decision, the exact tree
    (FNV of tree_signature) and the search statistics — disc and polygon
    scenes alike."""
    c, st = golden_io.cases()[idx]
    d = c["decision"]
    cfg = ParallelConfig(rng_seed=int(c["seed"]))
    r = run_pmbs(st, cfg, ctx=ctx)
    assert r.stop_reason == d["stop"]
    assert r.iterations == d["iterations"] and r.expansions == d["expansions"]
    assert r.final_tree_depth == d["final_tree_depth"]
    assert list(r.action) == d["action"]
    assert r.signature_fnv == int(d["sig_fnv"])


def test_run_pmbs_budget_and_errors(ctx):
    from paper_2207_06649_b200.world import WorldState
    giant = WorldState.from_objects([{"kind": "disc", "radius": 0.2, "pose": [0.0, 0.0, 0.0]}])
    with pytest.raises(SearchError):
        run_pmbs(giant, ParallelConfig(), ctx=ctx)
    c, st = golden_io.cases()[17]
    r = run_pmbs(st, ParallelConfig(budget=Budget.iterations(3), rng_seed=5), ctx=ctx)
    assert r.iterations == 3 and r.stop_reason == "budget"


def _ctx_with(**env):
    """A context created under kernel-selection overrides: PPG_FORCE_GENERIC=1
    (straight transcription), PPG_WARP_MAX=0 (no warp-per-env latency mode)."""
    import os
    from paper_2207_06649_b200 import Context
    old = {k: os.environ.get(k) for k in env}
    os.environ.update({k: str(v) for k, v in env.items()})
    try:
        return Context(0, default_params())
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v


def _generic_ctx():
    return _ctx_with(PPG_FORCE_GENERIC=1)


MODES = {"warp": {}, "lane": {"PPG_WARP_MAX": 0}, "generic": {"PPG_FORCE_GENERIC": 1},
         "hybrid": {"PPG_HYBRID_MIN": 0},  # hybrid: warp sampler / grasp + lane physics lockstep rounds
         "nofix": {"PPG_NO_FIXPOINT": 1}}  # no fixed-point substep skipping (must not change a bit)


@pytest.mark.parametrize("n,motif", [(1, "random"), (3, "random"), (6, "random"), (8, "random"), (9, "random"),
                                     (11, "random"), (12, "ring"), (14, "ring"), (16, "ring"), (20, "ring")])
def test_disc_fast_path_matches_generic_and_oracle(ctx, n, motif):
    """resolve_disc.cu (register-resident persistent kernel, object counts
    <= 16) against the straight transcription and the CPU oracle, bitwise,
    on all sampled pushes of several scenes (so start collisions, empty
    contacts, deep clusters and non-convergence all occur)."""
    from paper_2207_06649_b200.scenes import _take, generate_cases
    t, poses, ok = generate_cases(n, np.arange(4000, 4024), 0.0, motif)
    sel = np.nonzero(ok)[0][:12]
    t, poses = _take(t, sel), poses[sel]
    ctx.set_params(P)
    cand, cnt = ctx.sample_pushes_arrays(poses, t)
    idx = np.concatenate([np.full(c, k) for k, c in enumerate(cnt)]).astype(np.int64)
    pushes = np.concatenate([cand[k, :c] for k, c in enumerate(cnt)])
    # add start-collision pushes (tip placed on each scene's target)
    bad = np.stack([[p[0, 0], p[0, 1], p[0, 0] + 0.05, p[0, 1]] for p in poses])
    idx = np.concatenate([idx, np.arange(len(poses))])
    pushes = np.concatenate([pushes, bad])
    tt = _take(t, idx)
    pp = np.ascontiguousarray(poses[idx])
    o3, s3, r3 = port.batch_resolve(tt, pp, pushes, P)
    assert np.all(s3[-len(poses):] == 1)
    for mode, env in MODES.items():
        c = _ctx_with(**env)
        out, st, res = c.batch_resolve_arrays(tt, pp, pushes)
        c.close()
        assert np.array_equal(st, s3), mode
        assert _bitwise(out, o3).all(), mode
        assert np.array_equal(res.view(np.uint64), r3.view(np.uint64)), mode


@pytest.mark.parametrize("mode", list(MODES))
def test_all_kernel_modes_on_golden_resolve_sets(mode):
    c = _ctx_with(**MODES[mode])
    for name in ["discs", "ring16", "hard18"]:
        t, poses, pushes, status, digests, out_ref = golden_io.resolve_set(name)
        out, st, resid = c.batch_resolve_arrays(t, poses, pushes)
        assert np.array_equal(st, status), (mode, name)
        ok = status == 0
        assert _bitwise(out[ok], out_ref[ok]).all(), (mode, name)
    c.close()


@pytest.mark.parametrize("mode", ["warp", "lane", "hybrid", "nofix"])
def test_simulate_and_expand_modes(mode):
    c = _ctx_with(**MODES[mode])
    cases = {cc["case_id"]: st for cc, st in golden_io.cases()}
    for cid, ne, seed, cap, poses, meta, rewards in golden_io.simulate_sets():
        st = cases[cid]
        if not np.all(st.kind == 0):
            continue
        c.set_params(default_params(n_envs=ne, rng_seed=seed))
        c.set_scene(st)
        r, ctr = c.simulate_arrays(poses, meta, ne, True, seed, 0, cap)
        assert np.array_equal(r, rewards), (mode, cid)
        ro, co = port.simulate(st, poses, meta, ne, True, seed, 0, cap, default_params(n_envs=ne))
        assert np.array_equal(ctr, co), (mode, cid)
    c.set_params(P)
    for cc, st in golden_io.cases()[10:13]:
        c.set_scene(st)
        sp = port.sample_pushes(st, P)
        parents = np.repeat(st.poses[None], len(sp), 0)
        child, status, g, nu, un = c.expand_arrays(parents, sp)
        exp, est, _ = port.batch_resolve(ShapeTable.shared(st), parents, sp, P)
        assert np.array_equal(status, est), mode
        for k in range(len(sp)):
            if est[k] == 0:
                s2 = st.with_poses(exp[k])
                sp2 = port.sample_pushes(s2, P)
                assert nu[k] == len(sp2) and _bitwise(un[k, :nu[k]][None], sp2[None]).all(), mode
                assert bool(g[k]) == port.graspable(s2, P)[0], mode
    c.close()


@pytest.mark.parametrize("env", [{"PPG_WARP_MAX": 0}, {"PPG_HYBRID_MIN": 0}])
@pytest.mark.parametrize("idx", [12, 17, 19])
def test_fingerprints_lane_mode(idx, env):
    c = _ctx_with(**env)
    cc, st = golden_io.cases()[idx]
    d = cc["decision"]
    r = run_pmbs(st, ParallelConfig(rng_seed=int(cc["seed"])), ctx=c)
    assert list(r.action) == d["action"] and r.signature_fnv == int(d["sig_fnv"])
    c.close()


@pytest.mark.parametrize("shards", [1, 2, 3])
def test_device_shards_reproduce_unsharded_lockstep(shards):
    """The multi-GPU lockstep driver with `shards` device shards emulated in
    one process (separate contexts on cuda:0, host-mediated exchange) equals
    the reference batch_simulate goldens bit for bit."""
    from paper_2207_06649_b200.sharded import DeviceShard, InProcessComm, env_range, sharded_simulate
    cases = {cc["case_id"]: st for cc, st in golden_io.cases()}
    ctxs = [_ctx_with() for _ in range(shards)]
    for cid, ne, seed, cap, poses, meta, rewards in golden_io.simulate_sets():
        st = cases[cid]
        for c in ctxs:
            c.set_params(default_params(n_envs=ne, rng_seed=seed))
            c.set_scene(st)
        ranges = [env_range(ne, shards, r) for r in range(shards)]
        r, ctr = sharded_simulate([DeviceShard(c) for c in ctxs], InProcessComm(), poses, meta, ne, True, seed, 0,
                                  cap, ranges)
        assert np.array_equal(r, rewards), (shards, cid)
        ro, co = port.simulate(st, poses, meta, ne, True, seed, 0, cap, default_params(n_envs=ne))
        assert ctr[0] == co[0] and ctr[3] == co[3] and ctr[1] == co[1], (shards, cid)
    for c in ctxs:
        c.close()


@pytest.mark.parametrize("planner,shards", [("host", 1), ("device", 1), ("device", 3), ("host", 2)])
def test_run_pmbs_through_sharded_hook(planner, shards):
    """ppg_run_pmbs with the sharded simulate hook (`shards` ranks emulated in
    one process) reproduces the reference fingerprint, with the tree on the
    host or on the device: the multi-GPU planner path is the same algorithm."""
    from paper_2207_06649_b200.sharded import InProcessComm, ShardedSimulateHook
    ctxs = [_ctx_with() for _ in range(shards)]
    cc, st = golden_io.cases()[12]
    d = cc["decision"]
    cfg = ParallelConfig(rng_seed=int(cc["seed"]))
    for c in ctxs:
        c.set_params(cfg.to_params())
        c.set_scene(st)
    c = ctxs[0]
    c.set_planner(planner)
    hook = ShardedSimulateHook(c, InProcessComm(), shards, 0, extra_ctxs=ctxs[1:])
    r = run_pmbs(st, cfg, ctx=c, want_signature=True)
    hook.remove()
    assert hook.error is None
    assert list(r.action) == d["action"] and r.signature_fnv == int(d["sig_fnv"])
    r2 = run_pmbs(st, cfg, ctx=c, want_signature=True)  # the hook removed: built-in lockstep, same tree
    assert r2.signature == r.signature
    assert (r2.env_steps, r2.rollout_steps, r2.lockstep_rounds) == (r.env_steps, r.rollout_steps, r.lockstep_rounds)
    for x in ctxs:
        x.close()


def test_device_tree_sharded_hook_wide():
    """Device tree + 2 emulated shards on a wide batch (N_e = 2,000, dense
    ring): same tree and counters as the unsharded device tree."""
    from paper_2207_06649_b200.scenes import generate_case
    from paper_2207_06649_b200.sharded import InProcessComm, ShardedSimulateHook
    st = generate_case(16, 0.0, 3, "ring")
    cfg = ParallelConfig(rng_seed=3, n_envs=2000, budget=Budget.iterations(3))
    ctxs = [_ctx_with() for _ in range(2)]
    for c in ctxs:
        c.set_params(cfg.to_params())
        c.set_scene(st)
    base = run_pmbs(st, cfg, ctx=ctxs[0], want_signature=True)
    hook = ShardedSimulateHook(ctxs[0], InProcessComm(), 2, 0, extra_ctxs=ctxs[1:])
    r = run_pmbs(st, cfg, ctx=ctxs[0], want_signature=True)
    hook.remove()
    assert hook.error is None
    assert r.signature == base.signature and list(r.action) == list(base.action)
    assert (r.env_steps, r.rollout_steps, r.lockstep_rounds) == (base.env_steps, base.rollout_steps,
                                                                 base.lockstep_rounds)
    for c in ctxs:
        c.close()


def test_device_sincos_matches_glibc(ctx):
    """csrc/glibc_sincos.cuh vs the host libm sincos (the function the
    reference's Vec2::rotated calls, world.cpp:57-62), bitwise, on object
    angles [-pi, pi), every branch boundary and the wider reduction range."""
    import ctypes
    libm = ctypes.CDLL("libm.so.6")
    libm.sincos.argtypes = [ctypes.c_double, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
    rng = np.random.default_rng(5)
    xs = [rng.uniform(-np.pi, np.pi, 200000), rng.uniform(-1e4, 1e4, 20000), rng.uniform(-1e-6, 1e-6, 2000),
          rng.uniform(-0.2, 0.2, 20000)]
    edges = []
    for k in (0x3e400000, 0x3feb6000, 0x400368fd, 0x3fc020c4):  # branch thresholds (high words) and ~0.126
        for d in range(-3, 4):
            edges.append(np.array([(k << 32) + d * 977], np.uint64).view(np.float64)[0])
    edges += [0.0, -0.0, np.pi, -np.pi, np.pi / 2, -np.pi / 2, 2.426265, 0.855469, 1e-300, 1e-9]
    x = np.ascontiguousarray(np.concatenate(xs + [np.array(edges), -np.array(edges)]))
    s = np.empty_like(x)
    c = np.empty_like(x)
    assert ctx.lib.ppg_debug_sincos(ctx.ptr, x.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), len(x),
                                    s.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                    c.ctypes.data_as(ctypes.POINTER(ctypes.c_double))) == 0
    hs = np.empty_like(x)
    hc = np.empty_like(x)
    a, b = ctypes.c_double(), ctypes.c_double()
    for i, v in enumerate(x):
        libm.sincos(float(v), ctypes.byref(a), ctypes.byref(b))
        hs[i], hc[i] = a.value, b.value
    bad = np.nonzero((s.view(np.uint64) != hs.view(np.uint64)) | (c.view(np.uint64) != hc.view(np.uint64)))[0]
    assert len(bad) == 0, [(float(x[i]), float(s[i]), float(hs[i]), float(c[i]), float(hc[i])) for i in bad[:5]]


@pytest.mark.parametrize("n,pf,motif", [(3, 1.0, "random"), (6, 0.5, "random"), (9, 0.35, "random"),
                                        (10, 1.0, "random"), (12, 0.5, "wall"), (16, 0.35, "ring"),
                                        (16, 1.0, "random")])
def test_polygon_latency_mode_matches_generic_and_oracle(ctx, n, pf, motif):
    """warp_poly.cuh (one warp per env, SAT axes / closest-point edges /
    vertex updates spread over lanes, cached world polygons) against the
    straight one-lane transcription and the CPU oracle, bitwise, on every
    sampled push of several polygon scenes plus start-collision pushes."""
    from paper_2207_06649_b200.scenes import _take, generate_cases
    t, poses, ok = generate_cases(n, np.arange(7000, 7030), pf, motif)
    sel = np.nonzero(ok)[0][:10]
    if len(sel) == 0:
        pytest.skip("generator rejected every seed")
    t, poses = _take(t, sel), poses[sel]
    ctx.set_params(P)
    cand, cnt = ctx.sample_pushes_arrays(poses, t)
    idx = np.concatenate([np.full(c, k) for k, c in enumerate(cnt)]).astype(np.int64)
    pushes = np.concatenate([cand[k, :c] for k, c in enumerate(cnt)])
    bad = np.stack([[p[0, 0], p[0, 1], p[0, 0] + 0.05, p[0, 1]] for p in poses])
    idx = np.concatenate([idx, np.arange(len(poses))])
    pushes = np.concatenate([pushes, bad])
    tt = _take(t, idx)
    pp = np.ascontiguousarray(poses[idx])
    o3, s3, r3 = port.batch_resolve(tt, pp, pushes, P)
    for mode, env in [("warp", {}), ("generic", {"PPG_FORCE_GENERIC": 1})]:
        c = _ctx_with(**env)
        out, st, res = c.batch_resolve_arrays(tt, pp, pushes)
        c.close()
        assert np.array_equal(st, s3), mode
        assert _bitwise(out, o3).all(), mode
        assert np.array_equal(res.view(np.uint64), r3.view(np.uint64)), mode


@pytest.mark.parametrize("mode", ["warp", "generic"])
def test_polygon_golden_resolve_set_all_modes(mode):
    c = _ctx_with(**({"PPG_FORCE_GENERIC": 1} if mode == "generic" else {}))
    t, poses, pushes, status, digests, out_ref = golden_io.resolve_set("polygons")
    out, st, resid = c.batch_resolve_arrays(t, poses, pushes)
    assert np.array_equal(st, status)
    ok = status == 0
    assert _bitwise(out[ok], out_ref[ok]).all()
    c.close()


@pytest.mark.parametrize("idx", [8, 9, 15, 16])
def test_polygon_fingerprints_generic_vs_latency(idx):
    """The polygon proj/cases first decisions with the polygon latency mode
    switched off (PPG_WARP_POLY=0 -> one-lane kernels) match the fingerprint
    too, so both paths are pinned to the reference tree."""
    c = _ctx_with(PPG_WARP_POLY=0)
    cc, st = golden_io.cases()[idx]
    d = cc["decision"]
    r = run_pmbs(st, ParallelConfig(rng_seed=int(cc["seed"])), ctx=c)
    assert list(r.action) == d["action"] and r.signature_fnv == int(d["sig_fnv"])
    c.close()


def test_pipelined_host_batch_resolve(ctx):
    """ppg_batch_resolve with host buffers at E >= 32K runs as 4 slices on
    separate streams (copies overlap physics); results are element-wise, so
    they must equal the oracle bit for bit (checked on a 4K subsample spread
    over all slices) and be identical run to run."""
    from paper_2207_06649_b200.scenes import _take, c2_workload
    ctx.set_params(P)
    table, poses, pushes, _ = c2_workload(ctx, 40000)
    out, st, res = ctx.batch_resolve_arrays(table, poses, pushes)
    out2, st2, res2 = ctx.batch_resolve_arrays(table, poses, pushes)
    assert _bitwise(out, out2).all() and np.array_equal(st, st2)
    idx = np.linspace(0, 39999, 4000).astype(np.int64)
    o3, s3, r3 = port.batch_resolve(_take(table, idx), np.ascontiguousarray(poses[idx]),
                                    np.ascontiguousarray(pushes[idx]), P)
    assert np.array_equal(st[idx], s3)
    ok = s3 == 0
    assert _bitwise(out[idx][ok], o3[ok]).all()
    assert np.array_equal(res[idx].view(np.uint64), r3.view(np.uint64))


@pytest.mark.gpu
def test_streamed_host_batch_resolve_equals_chunked(ctx, monkeypatch):
    """Disc batches with host buffers (E >= 32K) run streamed: one physics
    launch overlapping the slice copies, synchronised by stream memory
    operations (ready flags / done counters).  Ragged E, start collisions
    (status 1) and every slice boundary: identical to the 4-slice chunked
    path (PPG_STREAMED=0) and to the oracle on a subsample."""
    from paper_2207_06649_b200 import Context
    from paper_2207_06649_b200.scenes import _take, c2_workload
    E = 40003
    ctx.set_params(P)
    table, poses, pushes, _ = c2_workload(ctx, E)
    pushes = pushes.copy()
    hit = np.arange(7, E, 997)
    pushes[hit, 0:2] = poses[hit, 0, 0:2]  # tip starts inside object 0: status 1
    pushes[hit, 2:4] = poses[hit, 0, 0:2] + 0.05
    out, st, res = ctx.batch_resolve_arrays(table, poses, pushes)
    assert (st[hit] == 1).all()
    monkeypatch.setenv("PPG_STREAMED", "0")
    c2 = Context(0, P)
    try:
        o2, s2, r2 = c2.batch_resolve_arrays(table, poses, pushes)
    finally:
        c2.close()
    assert np.array_equal(st, s2)
    assert _bitwise(out, o2).all()
    assert np.array_equal(res.view(np.uint64), r2.view(np.uint64))
    # pinned output buffers: the kernel writes results straight to host memory
    import torch
    po = torch.empty(poses.shape, dtype=torch.float64).pin_memory().numpy()
    ps = torch.full((E,), -7, dtype=torch.int32).pin_memory().numpy()
    pr = torch.full((E,), np.nan, dtype=torch.float64).pin_memory().numpy()
    po[:] = np.nan
    for _ in range(2):  # twice: the second call re-uses every buffer (epochs, counters)
        ctx.batch_resolve_arrays(table, poses, pushes, out=(po, ps, pr))
        assert np.array_equal(st, ps)
        assert _bitwise(out, po).all()
        assert np.array_equal(res.view(np.uint64), pr.view(np.uint64))
        po[:] = np.nan
    idx = np.unique(np.concatenate([np.linspace(0, E - 1, 2000).astype(np.int64), hit]))
    o3, s3, r3 = port.batch_resolve(_take(table, idx), np.ascontiguousarray(poses[idx]),
                                    np.ascontiguousarray(pushes[idx]), P)
    assert np.array_equal(st[idx], s3)
    ok = s3 == 0
    assert _bitwise(out[idx][ok], o3[ok]).all()


@pytest.mark.parametrize("n", [2, 5, 10, 13, 16])
def test_disc_kernel_walls_and_wild_inputs(n):
    """The lane kernel's float broad-phase filters and conservative clamp test
    on inputs the scene generator never makes: objects overlapping each other,
    at / beyond the walls (clamped on the first iteration), pushes into the
    walls, pushes starting far outside the workspace (the per-env margin
    scales with the largest coordinate) and zero-length pushes — bitwise
    against the oracle in lane, latency and generic mode."""
    rng = np.random.default_rng(100 + n)
    E = 2500
    h = 0.144
    poses = np.zeros((E, n, 3))
    poses[:, :, 0:2] = rng.uniform(-1.15 * h, 1.15 * h, (E, n, 2))
    poses[:, :, 2] = rng.uniform(-3.1, 3.1, (E, n))
    wall = rng.random((E, n)) < 0.3  # snap to a wall
    poses[:, :, 0] = np.where(wall, np.sign(poses[:, :, 0]) * (h - 1e-9 - rng.uniform(0, 2e-4, (E, n))), poses[:, :, 0])
    radius = rng.uniform(0.008, 0.03, (E, n))
    ang = rng.uniform(-np.pi, np.pi, E)
    start = rng.uniform(-h, h, (E, 2))
    far = rng.random(E) < 0.05
    start[far] *= 40.0
    length = np.where(rng.random(E) < 0.05, 0.0, rng.uniform(0.01, 0.08, E))
    end = start + length[:, None] * np.stack([np.cos(ang), np.sin(ang)], 1)
    pushes = np.ascontiguousarray(np.concatenate([start, end], 1))
    t = ShapeTable(np.zeros((E, n), np.int32), np.ascontiguousarray(radius), np.zeros((E, n), np.int32),
                   np.zeros((E, n, 8, 2)), np.zeros(E, np.int32), 0.288, 0.0, n, E)
    o3, s3, r3 = port.batch_resolve(t, poses, pushes, P)
    for mode in ("lane", "warp", "generic"):
        c = _ctx_with(**MODES[mode])
        out, st, res = c.batch_resolve_arrays(t, poses, pushes)
        c.close()
        assert np.array_equal(st, s3), mode
        assert _bitwise(out, o3).all(), mode
        assert np.array_equal(res.view(np.uint64), r3.view(np.uint64)), mode


@pytest.mark.parametrize("n", [16, 20])
def test_streamed_zero_copy_large_object_counts(n, monkeypatch):
    """Streamed + zero-copy output with records longer than a warp (3n > 32
    doubles per env; n > 14 has no theta plane, so theta is re-read from the
    device input): identical to the chunked path, pinned outputs, 33K envs of
    random clutter (walls, overlaps, start collisions)."""
    import torch
    from paper_2207_06649_b200 import Context
    rng = np.random.default_rng(7 + n)
    E, h = 33003, 0.144
    poses = np.zeros((E, n, 3))
    poses[:, :, 0:2] = rng.uniform(-h, h, (E, n, 2))
    poses[:, :, 2] = rng.uniform(-3.1, 3.1, (E, n))
    radius = rng.uniform(0.006, 0.016, (E, n))
    ang = rng.uniform(-np.pi, np.pi, E)
    start = rng.uniform(-0.12, 0.12, (E, 2))
    end = start + 0.05 * np.stack([np.cos(ang), np.sin(ang)], 1)
    pushes = np.ascontiguousarray(np.concatenate([start, end], 1))
    t = ShapeTable(np.zeros((E, n), np.int32), np.ascontiguousarray(radius), np.zeros((E, n), np.int32),
                   np.zeros((E, n, 8, 2)), np.zeros(E, np.int32), 0.288, 0.0, n, E)
    c1 = Context(0, P)
    po = torch.empty(poses.shape, dtype=torch.float64).pin_memory().numpy()
    ps = torch.empty((E,), dtype=torch.int32).pin_memory().numpy()
    pr = torch.empty((E,), dtype=torch.float64).pin_memory().numpy()
    c1.batch_resolve_arrays(t, poses, pushes, out=(po, ps, pr))
    c1.close()
    monkeypatch.setenv("PPG_STREAMED", "0")
    c2 = Context(0, P)
    o2, s2, r2 = c2.batch_resolve_arrays(t, poses, pushes)
    c2.close()
    assert len(np.unique(s2)) >= 2
    assert np.array_equal(ps, s2)
    assert _bitwise(po, o2).all()
    assert np.array_equal(pr.view(np.uint64), r2.view(np.uint64))


@pytest.mark.gpu
@pytest.mark.parametrize("pattern", ["all", "tail", "every_other"])
def test_streamed_zero_copy_start_collisions(ctx, pattern):
    """Zero-copy (pinned) outputs when whole warps only see start collisions
    (status 1, found during env init): every env's record must be written —
    pinned buffers pre-filled with sentinels, compared with the chunked path
    (PPG_STREAMED=0) and the oracle.  `all`: every push starts inside object
    0; `tail`: the last 3,000 envs do (the warps that drain the batch);
    `every_other`: alternate envs do."""
    import torch
    from paper_2207_06649_b200 import Context
    from paper_2207_06649_b200.scenes import _take, c2_workload
    E = 36011
    ctx.set_params(P)
    table, poses, pushes, _ = c2_workload(ctx, E)
    pushes = pushes.copy()
    hit = {"all": np.arange(E), "tail": np.arange(E - 3000, E), "every_other": np.arange(0, E, 2)}[pattern]
    pushes[hit, 0:2] = poses[hit, 0, 0:2]
    pushes[hit, 2:4] = poses[hit, 0, 0:2] + 0.05
    po = torch.empty(poses.shape, dtype=torch.float64).pin_memory().numpy()
    ps = torch.full((E,), -7, dtype=torch.int32).pin_memory().numpy()
    pr = torch.empty((E,), dtype=torch.float64).pin_memory().numpy()
    for _ in range(2):
        po[:] = np.nan
        ps[:] = -7
        pr[:] = np.nan
        ctx.batch_resolve_arrays(table, poses, pushes, out=(po, ps, pr))
        assert (ps[hit] == 1).all()
        assert (ps >= 0).all() and not np.isnan(pr).any() and not np.isnan(po).any()
    import os
    os.environ["PPG_STREAMED"] = "0"
    try:
        c2 = Context(0, P)
        o2, s2, r2 = c2.batch_resolve_arrays(table, poses, pushes)
        c2.close()
    finally:
        os.environ.pop("PPG_STREAMED", None)
    assert np.array_equal(ps, s2)
    assert _bitwise(po, o2).all()
    assert np.array_equal(pr.view(np.uint64), r2.view(np.uint64))
    idx = np.unique(np.concatenate([np.linspace(0, E - 1, 1500).astype(np.int64), hit[-200:]]))
    o3, s3, r3 = port.batch_resolve(_take(table, idx), np.ascontiguousarray(poses[idx]),
                                    np.ascontiguousarray(pushes[idx]), P)
    assert np.array_equal(ps[idx], s3)
    assert _bitwise(po[idx], o3).all()


@pytest.mark.gpu
def test_simulate_count_same_trajectory(ctx):
    """ppg_simulate_count (the rollout roofline numerator) runs the same
    rollouts: rewards-defining counters equal ppg_simulate's; every rollout
    step contributes sample + resolve work and grasp work after a resolve."""
    cases = {c["case_id"]: s for c, s in golden_io.cases()}
    for cid, ne, seed, cap, nposes, meta, rewards in golden_io.simulate_sets():
        ctx.set_params(default_params(n_envs=ne, rng_seed=seed))
        ctx.set_scene(cases[cid])
        r, ctr = ctx.simulate_arrays(nposes, meta, ne, True, seed, 0, cap)
        ops, ctr2 = ctx.simulate_count_arrays(nposes, meta, ne, True, seed, 0, cap)
        assert np.array_equal(ctr, ctr2), cid
        if ctr[0] > 0:
            assert ops[1] >= 31 * ctr[0] * cases[cid].n * 16  # every candidate of every step
            assert ops[0] > 0 and ops[2] >= 150 * 16
