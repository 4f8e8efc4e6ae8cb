"""The C-ABI library loads on a host without a GPU, exports every symbol
include/pushplan_gpu.h declares, and fails loudly (no CPU fallback) when no
device is present."""
import ctypes
import os
import re

import pytest

from paper_2207_06649_b200 import abi

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "pushplan_gpu.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(ppg_[a-z_0-9]+)\s*\(", text)) - {"ppg_shapes"})


def test_header_and_binding_agree():
    assert declared_functions() == sorted(abi.SIGNATURES)


def test_library_exports_every_declared_symbol():
    lib = abi.load_library()
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_version_and_defaults():
    lib = abi.load_library()
    assert b"sm_100a" in lib.ppg_version()
    p = abi.PpgParams()
    lib.ppg_params_default(ctypes.byref(p))
    d = abi.default_params()
    for f, _ in abi.PpgParams._fields_:
        assert getattr(p, f) == getattr(d, f), f


def test_no_device_fails_loudly():
    lib = abi.load_library()
    if lib.ppg_device_count() > 0:
        pytest.skip("a GPU is present")
    err = ctypes.c_int()
    assert not lib.ppg_create(0, None, ctypes.byref(err))
    assert err.value == abi.PPG_ENODEVICE
    from paper_2207_06649_b200 import Context, DeviceError
    with pytest.raises(DeviceError):
        Context(0)


def test_state_digest_host_helper_matches_golden():
    import golden_io
    import numpy as np
    from paper_2207_06649_b200.world import ShapeTable
    lib = abi.load_library()
    for c, st in golden_io.cases():
        t = ShapeTable.shared(st)
        out = np.zeros(1, np.uint64)
        poses = np.ascontiguousarray(st.poses.reshape(1, st.n, 3))
        assert lib.ppg_state_digest(ctypes.byref(t.struct()), abi.dptr(poses), 1, abi.u64ptr(out)) == 0
        assert int(out[0]) == int(c["digest"])


def test_nccl_loaded_before_torch_is_torchs_build():
    """The library loads NCCL at run time; loaded before torch it must be the
    copy torch ships (a system libnccl.so.2 would shadow torch's by soname
    and break `import torch`).  Runs in a fresh interpreter."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys; sys.path.insert(0, %r)\n"
            "import paper_2207_06649_b200 as p\n"
            "assert len(p.nccl_unique_id()) == 128\n"
            "import torch, torch.distributed\n"
            "print('ok', torch.cuda.nccl.version())\n") % root
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.startswith("ok"), r.stderr[-2000:]
