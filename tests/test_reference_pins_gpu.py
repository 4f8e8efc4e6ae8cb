"""GPU results pinned directly to the unmodified reference (oracle/_ref) on
the configurations the bench measures (VERDICT r1 task 1):

* the FULL bench workload — BASELINE config 2, 65,536 generate_case(10)
  disc scenes with one keyed sampled push each — through the host C-ABI
  (streamed, zero-copy into pinned buffers) and the device-buffer API, every
  env's status and poses bit-identical to the reference batch_resolve
  (push_sim.cpp:132-152) run on the reference's own inputs;
* the polygon variant (ShapeMix{0.35}, 16,384 envs);
* the algorithmic-work counters behind the roofline numerator
  (ppg_batch_resolve_count_dev) against the instrumented C restatement;
* run_pmbs fingerprints at wide N_e (1,000 / 4,096 / 16,384), on the C4
  dense ring motifs and on polygon cases (tests/golden/wide.json, produced by
  the reference's run_pmbs).
The reference itself runs here only as the checker (tests may execute
oracle/); the GPU box has the prebuilt oracle/_ref."""
import ctypes

import numpy as np
import pytest

import golden_io
from oracle import port, ref
from paper_2207_06649_b200 import Budget, ParallelConfig, run_pmbs
from paper_2207_06649_b200.abi import default_params, dptr, u64ptr

pytestmark = pytest.mark.gpu
P = default_params()


def _need_ref():
    if not ref.available():
        pytest.skip("oracle/_ref not built")


def _digests(lib, table, poses):
    out = np.zeros(poses.shape[0], np.uint64)
    assert lib.ppg_state_digest(ctypes.byref(table.struct()), dptr(np.ascontiguousarray(poses)), poses.shape[0],
                                u64ptr(out)) == 0
    return out


@pytest.mark.parametrize("pf,E", [(0.0, 65536), (0.35, 16384)])
def test_full_c2_workload_bitwise_vs_reference(ctx, pf, E):
    import torch
    from paper_2207_06649_b200.scenes import c2_workload
    _need_ref()
    ctx.set_params(P)
    table, poses, pushes, seeds = c2_workload(ctx, E, 10, pf)
    h, rpushes, rseeds = ref.c2_workload(E, 10, pf)
    # the same inputs: the product's host generator == the reference's
    assert np.array_equal(seeds, rseeds)
    assert np.array_equal(pushes.view(np.uint64), rpushes.view(np.uint64))
    pb = ref.PreparedBatch(None, None, rpushes, P, handle=h)
    pb.run(8)
    rout, rst, rdig = pb.results(10)
    # host C-ABI, pinned outputs (the bench's e2e path), sentinel-filled
    po = torch.empty(poses.shape, dtype=torch.float64).pin_memory().numpy()
    ps = torch.full((E,), -7, dtype=torch.int32).pin_memory().numpy()
    pr = torch.empty((E,), dtype=torch.float64).pin_memory().numpy()
    po[:] = np.nan
    pr[:] = np.nan
    ctx.batch_resolve_arrays(table, poses, pushes, out=(po, ps, pr))
    assert np.array_equal(ps, rst)
    assert np.array_equal(po.view(np.uint64), rout.view(np.uint64))
    ok = rst == 0
    assert np.array_equal(_digests(ctx.lib, table, po)[ok], rdig[ok])
    # pageable outputs (copy-back path)
    o2, s2, r2 = ctx.batch_resolve_arrays(table, poses, pushes)
    assert np.array_equal(s2, rst) and np.array_equal(o2.view(np.uint64), rout.view(np.uint64))
    assert np.array_equal(r2.view(np.uint64), pr.view(np.uint64))


def test_work_counters_match_instrumented_oracle(ctx):
    """ppg_batch_resolve_count_dev (the roofline numerator's source) ==
    the instrumented C restatement's counters, env by env."""
    import torch
    from paper_2207_06649_b200.abi import PpgShapes
    from paper_2207_06649_b200.scenes import _take, c2_workload
    ctx.set_params(P)
    sets = []
    table, poses, pushes, _ = c2_workload(ctx, 65536)
    idx = np.linspace(0, 65535, 4096).astype(np.int64)
    sets.append((_take(table, idx), np.ascontiguousarray(poses[idx]), np.ascontiguousarray(pushes[idx])))
    for name in ("discs", "ring16", "hard18"):
        t, p, a, *_ = golden_io.resolve_set(name)
        sets.append((t, p, a))
    dev = torch.device("cuda", 0)
    for t, p, a in sets:
        E, n = p.shape[:2]
        _, _, _, cnt = port.batch_resolve(t, p, a, P, counts=True)
        d_kind = torch.from_numpy(t.kind).to(dev)
        d_rad = torch.from_numpy(t.radius).to(dev)
        d_tgt = torch.from_numpy(t.target_index).to(dev)
        d_p = torch.from_numpy(p).to(dev)
        d_a = torch.from_numpy(a).to(dev)
        d_c = torch.zeros((E, 8), dtype=torch.int64, device=dev)
        sh = PpgShapes(n, E, ctypes.cast(d_kind.data_ptr(), ctypes.POINTER(ctypes.c_int32)),
                       ctypes.cast(d_rad.data_ptr(), ctypes.POINTER(ctypes.c_double)), None, None,
                       ctypes.cast(d_tgt.data_ptr(), ctypes.POINTER(ctypes.c_int32)), 0.288, 0.0)
        rc = ctx.lib.ppg_batch_resolve_count_dev(ctx.ptr, ctypes.byref(sh), d_p.data_ptr(), d_a.data_ptr(), E,
                                                 d_c.data_ptr(), None)
        assert rc == 0
        torch.cuda.synchronize()
        assert np.array_equal(d_c.cpu().numpy(), cnt)


def _wide_cfg(rec):
    if rec["kind"] == "case":
        return ParallelConfig(rng_seed=int(rec["seed"]), n_envs=rec["n_envs"],
                              budget=Budget.iterations(rec["max_iterations"]))
    return ParallelConfig(rng_seed=int(rec["seed"]), n_envs=rec["n_envs"], tree_depth=rec["tree_depth"],
                          pushes_per_object=rec["pushes_per_object"], budget=Budget.iterations(rec["max_iterations"]))


def _wide_state(rec):
    if rec["kind"] == "case":
        return {c["case_id"]: s for c, s in golden_io.cases()}[rec["case_id"]]
    from paper_2207_06649_b200.scenes import generate_case
    return generate_case(rec["n_objects"], 0.0, rec["scene_seed"], "ring")


def _wide_ids():
    out = []
    for r in golden_io.wide():
        out.append(f"{r['case_id']}-{r['n_envs']}" if r["kind"] == "case"
                   else f"ring{r['n_objects']}-s{r['scene_seed']}-{r['n_envs']}")
    return out


@pytest.mark.parametrize("k", range(len(golden_io.wide())), ids=_wide_ids())
def test_wide_fingerprints_vs_reference(ctx, k):
    rec = golden_io.wide()[k]
    r = run_pmbs(_wide_state(rec), _wide_cfg(rec), ctx=ctx)
    d = rec["decision"]
    assert list(r.action) == d["action"]
    assert r.signature_fnv == int(d["sig_fnv"])
    assert (r.iterations, r.expansions, r.stop_reason, r.final_tree_depth) == \
        (d["iterations"], d["expansions"], d["stop"], d["final_tree_depth"])


@pytest.mark.parametrize("mode", [{"PPG_HYBRID_MIN": 0}, {"PPG_PLANNER": "host"}])
def test_wide_fingerprints_other_modes(mode):
    """Hybrid rounds everywhere and the host-tree planner on the same
    reference fingerprints (the N_e <= 4,096 entries)."""
    from test_gpu_parity import _ctx_with
    c = _ctx_with(**mode)
    try:
        for rec in golden_io.wide():
            if rec["n_envs"] > 4096:
                continue
            r = run_pmbs(_wide_state(rec), _wide_cfg(rec), ctx=c)
            assert r.signature_fnv == int(rec["decision"]["sig_fnv"]), (mode, rec)
    finally:
        c.close()
