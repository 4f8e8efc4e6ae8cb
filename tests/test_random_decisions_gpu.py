"""Randomised parity of whole PMBS decisions on the device tree (the
asynchronous lockstep with early, pending-bound and speculative re-purposing
decisions) against the unmodified reference (oracle/_ref, run_pmbs with a
WorkerPool): generated scenes of 6-16 objects — discs, polygon mixes and
all-polygon scenes; random, ring and wall motifs — at N_e 64 / 256 / 1000.
Action and tree signature (visits, q sums, structure) must be identical.
tools/stress_decisions.py runs the same check on more scenes."""
import os

import pytest

from oracle import ref
from paper_2207_06649_b200 import Context, ParallelConfig, run_pmbs
from paper_2207_06649_b200.scenes import generate_case

pytestmark = pytest.mark.gpu

CASES = [(6, 0.0, "random", 64), (10, 0.0, "ring", 256), (13, 0.35, "wall", 64), (8, 1.0, "random", 256),
         (16, 0.0, "random", 1000), (12, 0.35, "ring", 64), (9, 0.0, "wall", 1000), (11, 1.0, "ring", 64)]


@pytest.fixture(scope="module")
def ctx():
    c = Context(0)
    yield c
    c.close()


@pytest.mark.parametrize("k", range(len(CASES)))
def test_random_decision_matches_reference(ctx, k):
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    n, pf, motif, ne = CASES[k]
    seed = 5000 + 101 * k
    try:
        st = generate_case(n, pf, seed, motif)
    except RuntimeError:
        pytest.skip("generator rejected the seed")
    cfg = ParallelConfig(rng_seed=seed, n_envs=ne)
    q = ref.run_search(st, cfg.to_params(), threads=os.cpu_count() or 1)
    if q.get("rc", 0) != 0:
        with pytest.raises(Exception):
            run_pmbs(st, cfg, ctx=ctx)
        return
    r = run_pmbs(st, cfg, ctx=ctx)
    assert list(r.action) == list(q["action"])
    assert r.signature_fnv == q["sig_fnv"]
    assert (r.iterations, r.expansions) == (q["iterations"], q["expansions"])
