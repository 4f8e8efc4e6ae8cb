"""The reference's acceptance criteria as GPU parity gates:
C1 (acceptance.cpp:184-211) — PMBS with one environment and no leaf
parallelism equals the serial MCTS tree on 25 deep search cases x 500
iterations; C4 (:283-305) — N_e = 16 searches are scheduling-independent:
here, identical to the reference tree in every device kernel mode."""
import pytest

import golden_io
from paper_2207_06649_b200 import Budget, ParallelConfig, run_pmbs

pytestmark = pytest.mark.gpu


def test_c1_single_env_pmbs_equals_serial_mcts(ctx):
    for rec, st in golden_io.acceptance()["c1"]:
        cfg = ParallelConfig(budget=Budget.iterations(500), rng_seed=rec["seed"], n_envs=1, leaf_parallel=False)
        r = run_pmbs(st, cfg, ctx=ctx)
        assert r.signature_fnv == int(rec["sig_fnv"]), rec["seed"]
        assert list(r.action) == rec["action"] and r.iterations == rec["iterations"] and r.stop_reason == rec["stop"]


@pytest.mark.parametrize("mode", [{}, {"PPG_WARP_MAX": 0}, {"PPG_FORCE_GENERIC": 1}, {"PPG_HYBRID_MIN": 0}])
def test_c4_scheduling_independence(mode):
    from test_gpu_parity import _ctx_with
    c = _ctx_with(**mode)
    for rec, st in golden_io.acceptance()["c4"]:
        cfg = ParallelConfig(budget=Budget.iterations(200), rng_seed=rec["seed"], n_envs=16)
        r = run_pmbs(st, cfg, ctx=c)
        assert r.signature_fnv == int(rec["sig_fnv"]), (mode, rec["seed"])
        assert list(r.action) == rec["action"]
    c.close()
