"""sample_pushes / graspable one warp per state (sample_grasp_warp_kernel,
small batches) == one lane per state (sample_kernel / grasp_kernel, large
batches; PPG_SAMPLE_WARP_MAX=0 forces it), bit for bit: candidate lists and
counts on generated disc / polygon scenes, graspable flag, margin, best pose
and angle on jittered states of every proj/cases scene.  Both paths are
pinned to the reference elsewhere (tests/test_gpu_parity.py: the 20 cases'
sample FNVs and grasp poses run the warp path now)."""
import numpy as np
import pytest

import golden_io
from paper_2207_06649_b200 import Context
from paper_2207_06649_b200.scenes import generate_cases

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = Context(0)
    yield c
    c.close()


@pytest.mark.parametrize("pf", [0.0, 0.35, 1.0])
@pytest.mark.parametrize("n", [4, 10, 16])
def test_sample_pushes_warp_equals_lane(ctx, monkeypatch, pf, n):
    table, poses, ok = generate_cases(n, np.arange(5000, 5600, dtype=np.uint64), pf)
    sel = np.nonzero(ok)[0][:400]
    from paper_2207_06649_b200.scenes import _take
    table, poses = _take(table, sel), np.ascontiguousarray(poses[sel])
    monkeypatch.delenv("PPG_SAMPLE_WARP_MAX", raising=False)
    out_w, cnt_w = ctx.sample_pushes_arrays(poses, table)
    monkeypatch.setenv("PPG_SAMPLE_WARP_MAX", "0")
    out_l, cnt_l = ctx.sample_pushes_arrays(poses, table)
    assert np.array_equal(cnt_w, cnt_l)
    for e in range(len(sel)):
        k = cnt_l[e]
        assert np.array_equal(out_w[e, :k].view(np.uint64), out_l[e, :k].view(np.uint64)), e


def test_graspable_warp_equals_lane(ctx, monkeypatch):
    rng = np.random.default_rng(3)
    for cc, st in golden_io.cases():
        ctx.set_scene(st)
        base = np.asarray(st.poses, np.float64)
        poses = np.repeat(base[None], 64, axis=0)
        poses[1:, :, :2] += rng.normal(0.0, 0.01, size=(63, base.shape[0], 2))
        poses[1:, :, 2] += rng.normal(0.0, 0.3, size=(63, base.shape[0]))
        monkeypatch.delenv("PPG_SAMPLE_WARP_MAX", raising=False)
        w = ctx.graspable_arrays(poses)
        monkeypatch.setenv("PPG_SAMPLE_WARP_MAX", "0")
        l = ctx.graspable_arrays(poses)
        for a, b in zip(w, l):
            assert np.array_equal(np.asarray(a).view(np.uint8), np.asarray(b).view(np.uint8)), cc["case_id"]
