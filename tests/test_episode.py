"""Episode driver (paper_2207_06649_b200.episode, bench.cpp:54-126 restated
over the GPU planner): same action sequence, action count and outcome as
the reference's run_episode on proj/cases scenes, and the JSONL log it
writes verifies under the reference's own replay_log (bench.cpp:319-377)."""
import json
import os

import pytest

import golden_io
from oracle import ref
from paper_2207_06649_b200 import ParallelConfig
from paper_2207_06649_b200.episode import episode_seed, mix_keys, run_episode


def test_seeds_match_reference_fixtures():
    for c, _ in golden_io.cases():
        assert mix_keys(episode_seed(0, c["case_id"], 0), 0) == int(c["seed"])


@pytest.mark.gpu
@pytest.mark.parametrize("idx,trial", [(0, 0), (9, 1), (12, 0), (15, 2), (16, 0), (17, 0), (19, 3)])
def test_episode_equals_reference(ctx, tmp_path, idx, trial):
    c, st = golden_io.cases()[idx]
    cfg = ParallelConfig()
    seed = episode_seed(0, c["case_id"], trial)
    path = tmp_path / "mine.jsonl"
    with open(path, "w") as f:
        r = run_episode(st, c["case_id"], trial, cfg, seed, log=f, ctx=ctx)
    assert r.completed
    recs = [json.loads(line) for line in open(path)]
    pushes = [x for x in recs if x["type"] == "push"]
    assert len(pushes) + 1 == r.actions_used
    if not ref.available():
        return
    ok, report = ref.replay_log(str(path))  # the reference re-folds OUR log through ITS simulator
    assert ok, report
    rp = str(tmp_path / "ref.jsonl")
    q = ref.run_episode(st, c["case_id"], trial, cfg.to_params(), 1, 0, 16, rp)
    assert q["actions_used"] == r.actions_used and q["completed"] == r.completed
    theirs = [json.loads(line) for line in open(rp)]
    assert [x for x in theirs if x["type"] == "push"] == pushes
    assert [x for x in theirs if x["type"] == "grasp"] == [x for x in recs if x["type"] == "grasp"]
