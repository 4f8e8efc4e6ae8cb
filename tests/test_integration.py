"""The reference-side binding (integration/pushplan_gpu_backend.*) compiled
inside the reference code base (oracle/_ref/libpushplan_adapter.so): the
reference's own types and call sites routed through the C-ABI reproduce the
reference's results bit for bit (acceptance C8 style, acceptance.cpp:372-412;
run_pmbs decisions and tree signatures)."""
import ctypes
import json
import os

import numpy as np
import pytest

import golden_io

ADAPTER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                       "libpushplan_adapter.so")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.exists(ADAPTER), reason="adapter not built (needs /root/reference)")]


def _lib():
    L = ctypes.CDLL(ADAPTER)
    L.adapter_check_c8.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_long), ctypes.POINTER(ctypes.c_long)]
    L.adapter_check_pmbs.argtypes = [ctypes.c_char_p, ctypes.c_char_p] + [ctypes.POINTER(ctypes.c_int)] * 3
    return L


def test_adapter_batch_resolve_equals_reference_elementwise():
    L = _lib()
    pairs, bad = ctypes.c_long(), ctypes.c_long()
    assert L.adapter_check_c8(600, ctypes.byref(pairs), ctypes.byref(bad)) == 0
    assert pairs.value >= 600
    assert bad.value == 0


@pytest.mark.parametrize("idx", [0, 10, 12, 17])
def test_adapter_run_pmbs_equals_reference(tmp_path, idx):
    c, st = golden_io.cases()[idx]
    if not np.all(st.kind == 0):
        pytest.skip("polygon case: decisions only (see test_gpu_parity)")
    objs = [{"kind": "disc", "radius": float(st.radius[i]), "pose": [float(v) for v in st.poses[i]]}
            for i in range(st.n)]
    path = tmp_path / f"{c['case_id']}.json"
    path.write_text(json.dumps({"workspace": {"side_length": st.side_length}, "objects": objs,
                                "target_index": st.target_index}))
    L = _lib()
    a, s, t = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    assert L.adapter_check_pmbs(str(path).encode(), c["case_id"].encode(), ctypes.byref(a), ctypes.byref(s),
                                ctypes.byref(t)) == 0
    assert a.value == 1 and s.value == 1 and t.value == 1


ACCEPTANCE = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                          "acceptance_gpu")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(ACCEPTANCE), reason="acceptance_gpu not built (needs /root/reference)")
@pytest.mark.parametrize("criterion", [1, 2, 3, 4, 8, 9])
def test_reference_acceptance_binary_on_the_gpu_core(criterion):
    """The reference's UNCHANGED acceptance suite (proj/tests/acceptance.cpp)
    linked against pushplan_core_gpu — the reference core whose
    batch_resolve and pmbs::run_pmbs are the device path (oracle/Makefile
    core_gpu): C1 (N_e = 1 PMBS tree == serial MCTS tree, via
    SearchResult::tree rebuilt from the device tree), C4 (identical trees
    across pool sizes), C8 (GPU batch_resolve == the reference resolve_push,
    bitwise digests), C2 / C3 / C9 on the reference functions it still uses."""
    import subprocess
    r = subprocess.run([ACCEPTANCE, "--criterion", str(criterion)], capture_output=True, text=True, timeout=1200)
    line = [ln for ln in r.stdout.splitlines() if ln.startswith(f"criterion {criterion}:")]
    assert line and ": PASS" in line[0], (r.stdout[-2000:], r.stderr[-2000:])
