"""The multi-GPU lockstep exchange over a real NCCL communicator on the device.

The gloo tests (test_sharded.py) cover world_size 2 on CPU and the emulated
device shards (test_gpu_parity.py) cover the device side with a host-mediated
exchange; this one runs `TorchComm` on an NCCL process group (world_size 1:
one GPU is all a round-end box has) so the record all-gather and the W
all-reduce go through NCCL on cuda:0, and checks the reference goldens
(pmbs.cpp:133-234 batch_simulate; pmbs.cpp:242-292 run_pmbs) bit for bit.
"""
import socket

import numpy as np
import pytest

import golden_io
from paper_2207_06649_b200 import Context, ParallelConfig, default_params, run_pmbs

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl_group():
    import torch
    import torch.distributed as dist
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1,
                            device_id=dev)
    assert dist.get_backend() == "nccl"
    yield dev
    dist.destroy_process_group()


def test_nccl_sharded_simulate_matches_goldens(nccl_group):
    from paper_2207_06649_b200.sharded import DeviceShard, TorchComm, env_range, sharded_simulate
    comm = TorchComm(device=nccl_group)
    cases = {cc["case_id"]: st for cc, st in golden_io.cases()}
    ctx = Context()
    n = 0
    for cid, ne, seed, cap, poses, meta, rewards in golden_io.simulate_sets():
        ctx.set_params(default_params(n_envs=ne, rng_seed=seed))
        ctx.set_scene(cases[cid])
        r, _ = sharded_simulate([DeviceShard(ctx)], comm, poses, meta, ne, True, seed, 0, cap,
                                [env_range(ne, 1, 0)])
        assert np.array_equal(r, rewards), cid
        n += 1
    ctx.close()
    assert n > 0


def test_nccl_run_pmbs_through_sharded_hook(nccl_group):
    from paper_2207_06649_b200.sharded import ShardedSimulateHook, TorchComm
    cc, st = golden_io.cases()[12]
    d = cc["decision"]
    cfg = ParallelConfig(rng_seed=int(cc["seed"]))
    ctx = Context()
    ctx.set_params(cfg.to_params())
    ctx.set_scene(st)
    ctx.set_planner("device")
    hook = ShardedSimulateHook(ctx, TorchComm(device=nccl_group), 1, 0)
    r = run_pmbs(st, cfg, ctx=ctx, want_signature=True)
    hook.remove()
    assert hook.error is None
    assert list(r.action) == d["action"] and r.signature_fnv == int(d["sig_fnv"])
    ctx.close()


def test_rank_context_library_native(nccl_group):
    """sharded.rank_context — the path bench.py's C5 block takes under
    torchrun: rank 0 makes the NCCL id, torch.distributed broadcasts it,
    ppg_create_rank builds the library's own communicator; run_pmbs on it
    (sharded device tree, in-library W all-reduce) == reference fingerprints."""
    from paper_2207_06649_b200.sharded import rank_context
    ctx = rank_context(0)
    try:
        assert ctx.shard_info() == {"rank": 0, "world": 1, "shards_here": 1, "transport": "nccl"}
        for idx in (4, 12, 17):
            cc, st = golden_io.cases()[idx]
            r = run_pmbs(st, ParallelConfig(rng_seed=int(cc["seed"])), ctx=ctx)
            assert list(r.action) == cc["decision"]["action"] and r.signature_fnv == int(cc["decision"]["sig_fnv"])
    finally:
        ctx.close()
