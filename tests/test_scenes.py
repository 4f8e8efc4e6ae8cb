"""Host input generators (paper_2207_06649_b200.scenes) against the reference
generator (oracle/_ref) and the golden fixtures: bit-identical scenes."""
import numpy as np
import pytest

import golden_io
from oracle import ref
from paper_2207_06649_b200 import scenes


def test_generate_matches_golden_resolve_sets():
    # resolve_discs.npz holds generate_case(10, {0.0}, 1000 + k) scenes in order
    t, poses, *_ = golden_io.resolve_set("discs")
    gt, gp, ok = scenes.generate_cases(10, np.arange(1000, 1000 + len(poses)), 0.0)
    assert ok.all()
    assert np.array_equal(gp.view(np.uint64), poses.view(np.uint64))
    assert np.array_equal(gt.radius.view(np.uint64), t.radius.view(np.uint64))


def test_generate_polygons_matches_golden():
    t, poses, *_ = golden_io.resolve_set("polygons")
    gt, gp, ok = scenes.generate_cases(10, np.arange(50000, 50000 + len(poses)), 0.35)
    assert ok.all()
    assert np.array_equal(gp.view(np.uint64), poses.view(np.uint64))
    assert np.array_equal(gt.vertices.view(np.uint64), t.vertices.view(np.uint64))
    assert np.array_equal(gt.kind, t.kind)


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("motif,n,pf", [("random", 8, 0.0), ("random", 12, 0.5), ("ring", 16, 0.0),
                                        ("ring", 18, 0.3), ("wall", 10, 0.2)])
def test_generate_matches_live_reference(motif, n, pf):
    seeds = np.arange(300, 360)
    gt, gp, ok = scenes.generate_cases(n, seeds, pf, motif)
    for i, s in enumerate(seeds):
        try:
            r = ref.generate_case(n, pf, int(s), scenes.MOTIFS[motif])
        except RuntimeError:
            assert not ok[i]
            continue
        assert ok[i]
        assert np.array_equal(gp[i].view(np.uint64), r.poses.view(np.uint64))
        assert np.array_equal(gt.kind[i], r.kind)
        assert np.array_equal(gt.vertices[i].view(np.uint64), r.vertices.view(np.uint64))


def test_keyed_picks_match_golden():
    for r in golden_io.rng():
        n = int(r["n"])
        if n > 2 ** 62:
            continue
        got = scenes.keyed_picks(int(r["seed"]), r["iter"], r["env"], [n])
        assert str(int(got[0])) == r["picks"][0]
