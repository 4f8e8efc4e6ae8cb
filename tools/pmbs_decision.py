"""One PMBS planning decision (run_pmbs) on 1..8 GPUs.

    python tools/pmbs_decision.py --case case_18 --n-envs 4096 --iters 5
    python -m torch.distributed.run --nproc-per-node 8 --master-addr 127.0.0.1 \
        tools/pmbs_decision.py --case case_18 --n-envs 65536 --iters 5

With WORLD_SIZE > 1 every rank runs the same host tree and the rollout batch
of each iteration is sharded by environment across the ranks
(paper_2207_06649_b200.sharded: one record allgather + one allreduce per
lockstep round over NCCL).  The decision, statistics and tree signature are
identical for every G (the env index -> RNG key map is global); rank 0
prints one JSON line.  Scenes: the committed proj/cases fixtures
(tests/golden/cases.json) or a dense ring motif (--motif-ring N, seed).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="case_18")
    ap.add_argument("--motif-ring", type=int, default=0, help="use generate_case_motif(Ring, N) instead")
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--n-envs", type=int, default=4096)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--tree-depth", type=int, default=7)
    ap.add_argument("--repeat", type=int, default=2)
    ap.add_argument("--planner", default="auto", choices=["auto", "host", "device"])
    args = ap.parse_args()

    import torch
    import torch.distributed as dist

    from paper_2207_06649_b200 import Budget, Context, ParallelConfig, run_pmbs
    from paper_2207_06649_b200.sharded import ShardedSimulateHook, TorchComm

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.motif_ring:
        from paper_2207_06649_b200.scenes import generate_case
        scene = generate_case(args.motif_ring, 0.0, args.seed, "ring")
        seed = args.seed
        name = f"ring{args.motif_ring}_s{args.seed}"
    else:
        import golden_io
        c, scene = {cc["case_id"]: (cc, st) for cc, st in golden_io.cases()}[args.case]
        seed = int(c["seed"])
        name = args.case
    ctx = Context(local)
    ctx.set_planner(args.planner)
    cfg = ParallelConfig(rng_seed=seed, n_envs=args.n_envs, tree_depth=args.tree_depth,
                         budget=Budget.iterations(args.iters))
    ctx.set_params(cfg.to_params())
    ctx.set_scene(scene)
    hook = ShardedSimulateHook(ctx, TorchComm(device=torch.device("cuda", local)), world, rank) if world > 1 else None
    best = None
    for _ in range(args.repeat):
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        r = run_pmbs(scene, cfg, ctx=ctx)
        dt = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([dt], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        best = dt if best is None else min(best, dt)
    if hook and hook.error:
        raise hook.error
    if rank == 0:
        print(json.dumps({"scene": name, "planner": args.planner, "n_gpus": world, "n_envs": args.n_envs, "iterations": r.iterations,
                          "expansions": r.expansions, "stop": r.stop_reason, "env_steps": r.env_steps,
                          "lockstep_rounds": r.lockstep_rounds, "s_per_decision": best,
                          "env_steps_per_s": r.env_steps / best, "action": list(r.action),
                          "tree_signature_fnv": hex(r.signature_fnv), "phase_s": r.phase_s}))
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
