"""The CPU oracle (oracle/pmbs_oracle.c) pinned against the reference: the
committed golden fixtures (always) and the compiled reference itself
(oracle/_ref, when present).  Bit-exact throughout."""
import numpy as np
import pytest

import golden_io
from oracle import port, ref
from paper_2207_06649_b200.abi import default_params
from paper_2207_06649_b200.world import ShapeTable

P = default_params()


@pytest.mark.parametrize("name", golden_io.RESOLVE_SETS)
def test_port_resolve_matches_golden(name):
    t, poses, pushes, status, digests, out_ref = golden_io.resolve_set(name)
    out, st, _ = port.batch_resolve(t, poses, pushes, P)
    assert np.array_equal(st, status)
    ok = status == 0
    assert np.array_equal(out[ok].view(np.uint64), out_ref[ok].view(np.uint64))
    assert np.array_equal(port.state_digests(t, out)[ok], digests[ok])


def test_port_cases_sample_grasp_digest():
    for c, st in golden_io.cases():
        assert port.state_digest(st) == int(c["digest"]), c["case_id"]
        sp = port.sample_pushes(st, P)
        assert len(sp) == c["n_pushes"]
        assert golden_io.fnv_bytes(sp.tobytes()) == int(c["pushes_fnv"]), c["case_id"]
        g = port.graspable(st, P)
        assert g[0] == c["graspable"] and g[1] == c["margin"] and [g[2], g[3], g[4]] == c["best"]


def test_port_rng_matches_golden():
    for r in golden_io.rng():
        picks = port.keyed_picks(int(r["seed"]), r["iter"], r["env"], 400, int(r["n"]))
        assert [str(v) for v in picks] == r["picks"]


def test_port_simulate_matches_golden():
    cases = {c["case_id"]: st for c, st in golden_io.cases()}
    for cid, ne, seed, cap, poses, meta, rewards in golden_io.simulate_sets():
        p = default_params(n_envs=ne, rng_seed=seed)
        r, ctr = port.simulate(cases[cid], poses, meta, ne, True, seed, 0, cap, p)
        assert np.array_equal(r, rewards), cid
        assert ctr[0] > 0


def test_port_lockstep_validation():
    cases = {c["case_id"]: st for c, st in golden_io.cases()}
    st = cases["case_13"]
    with pytest.raises(ValueError):
        port.simulate(st, np.repeat(st.poses[None], 5, 0), np.zeros((5, 3), np.int32), 4, True, 0, 0, 10, P)


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built (needs /root/reference)")
def test_port_matches_live_reference_random_scenes():
    states, pushes = [], []
    for k in range(120):
        s = ref.generate_case(9, 0.3, 777 + k)
        sp = ref.sample_pushes(s, P)
        assert np.array_equal(sp, port.sample_pushes(s, P))
        assert ref.graspable(s, P) == port.graspable(s, P)
        states.append(s)
        pushes.append(sp[int(ref.keyed_picks(3, k, 0, 1, len(sp))[0])])
    t = ShapeTable.per_env(states)
    poses = np.stack([s.poses for s in states])
    a = np.stack(pushes)
    o1, s1, d1, _ = ref.batch_resolve(t, poses, a, P)
    o2, s2, _ = port.batch_resolve(t, poses, a, P)
    assert np.array_equal(s1, s2)
    assert np.array_equal(o1.view(np.uint64), o2.view(np.uint64))
    for seed in (1, 99):
        assert np.array_equal(ref.keyed_picks(seed, 2, 3, 500, 37), port.keyed_picks(seed, 2, 3, 500, 37))
