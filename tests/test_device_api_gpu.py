"""ppg_batch_resolve_dev (device-resident inputs and shape tables) against the
host-buffer ppg_batch_resolve, bit for bit: disc batches on the warp path
(<= 2,048 envs), on the lane-per-env kernel reading the caller's [E][n]
radius table in place (> 2,048 envs; no shape-table transpose), and polygon
mixes (shape tables uploaded / transposed)."""
import ctypes

import numpy as np
import pytest
import torch

from paper_2207_06649_b200 import Context, default_params
from paper_2207_06649_b200.abi import PpgShapes
from paper_2207_06649_b200.scenes import c2_workload

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = Context(0, default_params())
    yield c
    c.close()


@pytest.mark.parametrize("E,pf", [(1024, 0.0), (6000, 0.0), (3000, 0.35)])
def test_device_api_equals_host_api(ctx, E, pf):
    table, poses, pushes, _ = c2_workload(ctx, E, 10, pf)
    h_out, h_st, h_res = ctx.batch_resolve_arrays(table, poses, pushes)
    dev = torch.device("cuda", 0)
    t = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev)
         for k, v in dict(p=poses, u=pushes, k=table.kind, r=table.radius, g=table.target_index,
                          nv=table.n_vertices, vt=table.vertices).items()}
    out = torch.full_like(t["p"], float("nan"))
    st = torch.full((E,), -7, dtype=torch.int32, device=dev)
    res = torch.full((E,), float("nan"), dtype=torch.float64, device=dev)
    P = ctypes.POINTER
    polys = pf > 0
    sh = PpgShapes(10, E, ctypes.cast(t["k"].data_ptr(), P(ctypes.c_int32)),
                   ctypes.cast(t["r"].data_ptr(), P(ctypes.c_double)),
                   ctypes.cast(t["nv"].data_ptr(), P(ctypes.c_int32)) if polys else None,
                   ctypes.cast(t["vt"].data_ptr(), P(ctypes.c_double)) if polys else None,
                   ctypes.cast(t["g"].data_ptr(), P(ctypes.c_int32)), 0.288, 0.0)
    stream = torch.cuda.current_stream(dev)
    rc = ctx.lib.ppg_batch_resolve_dev(ctx.ptr, ctypes.byref(sh), t["p"].data_ptr(), t["u"].data_ptr(), E,
                                       out.data_ptr(), st.data_ptr(), res.data_ptr(),
                                       ctypes.c_void_p(stream.cuda_stream))
    assert rc == 0, ctx.lib.ppg_last_error(ctx.ptr)
    torch.cuda.synchronize()
    assert np.array_equal(st.cpu().numpy(), h_st)
    assert np.array_equal(res.cpu().numpy().view(np.uint64), h_res.view(np.uint64))
    ok = h_st == 0
    assert np.array_equal(out.cpu().numpy()[ok].view(np.uint64), h_out[ok].view(np.uint64))
