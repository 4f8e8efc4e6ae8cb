"""Acceptance criterion 3 (reference acceptance.cpp:255-281) as a GPU gate:
the device select_batch (dt_select_kernel — the selection kernel inside
every PMBS iteration graph, pmbs.cpp:12-63) on 200 random explicit trees
must draw exactly the reference select_batch's (node, untried action) pairs
in the same order (hence unique pairs, the criterion), leave the same
virtual visits on every node, and reset_virtual must zero them (sum 0).
Fixture: tests/golden/c3_trees.npz, made by the reference itself
(make_golden.py c3 -> oracle/ref_shim.cpp ref_c3_trees)."""
import ctypes

import numpy as np
import pytest

import golden_io


def _device_select(ctx, a, t):
    lo, hi = int(a["node_off"][t]), int(a["node_off"][t + 1])
    N = hi - lo
    sl = {k: np.ascontiguousarray(a[k][lo:hi]) for k in ("parent", "depth", "visits", "q_sum", "flags",
                                                        "n_children", "n_untried")}
    ne = int(a["n_envs"][t])
    sn = np.zeros(ne, np.int32)
    su = np.zeros(ne, np.int32)
    nsel = ctypes.c_int32()
    vv = np.zeros(N, np.int64)
    vsum = ctypes.c_int64()
    rc = ctx.lib.ppg_debug_select_batch(ctx.ptr, N, *[sl[k].ctypes.data for k in ("parent", "depth", "visits", "q_sum",
                                                                              "flags", "n_children", "n_untried")],
                                        int(a["tree_depth"][t]), ne, 0.3, sn.ctypes.data, su.ctypes.data,
                                        ctypes.addressof(nsel), vv.ctypes.data, ctypes.addressof(vsum))
    assert rc == 0, ctx.lib.ppg_last_error(ctx.ptr)
    return sn[:nsel.value], su[:nsel.value], vv, vsum.value


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 1])
def test_c3_device_select_batch_matches_reference(ctx, variant):
    a = golden_io.c3_trees(variant)
    count = len(a["n_envs"])
    assert count == 200
    clean = 0
    for t in range(count):
        sn, su, vv, vsum = _device_select(ctx, a, t)
        plo, phi = int(a["pair_off"][t]), int(a["pair_off"][t + 1])
        lo, hi = int(a["node_off"][t]), int(a["node_off"][t + 1])
        assert np.array_equal(sn, a["sel_node"][plo:phi]), t
        assert np.array_equal(su, a["sel_untried"][plo:phi]), t
        assert np.array_equal(vv, a["vv"][lo:hi]), t
        assert vsum == 0 and int(a["vsum"][t]) == 0
        assert (len(sn) == 0) == bool(a["exhausted"][t])
        if len(set(zip(sn.tolist(), su.tolist()))) == len(sn) and len(sn) > 0:
            clean += 1
    assert clean == count  # the criterion: 200/200 invocations clean


def test_c3_fixture_is_the_reference():
    """(CPU) the committed fixture is what the reference produces now."""
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    for v in (0, 1):
        a = golden_io.c3_trees(v)
        b = ref.c3_trees(v)
        for k in a:
            assert np.array_equal(a[k], b[k]), (v, k)
