"""BASELINE configs[4], ZeRO-3 shaped: every rank all-gathers its shard of a 256 MB bf16
parameter tensor and reduce-scatters a 256 MB bf16 gradient tensor, with the staging pool
capped. Run under torchrun (one process per GPU):

  torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tools/zero3.py --caps 512,128,32

"256 MB" is the gathered parameter tensor (n shards of 256 MB / n) and the per-rank gradient
tensor (reduce-scattered to 256 MB / n per rank). Prints one JSON line per cap from rank 0.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--total-bytes", type=int, default=256 * 1000 * 1000)
    ap.add_argument("--caps", default="512,128,32", help="staging caps per rank, MiB")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--windows", action="store_true", help="register the four tensors as symmetric windows")
    ap.add_argument("--nccl", action="store_true", help="also time NCCL (NCCL_ALGO as set) on the same tensors")
    ap.add_argument("--group", action="store_true", help="issue each step's two calls as one group (one launch)")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    from paper_2506_20252_b200 import BFLOAT16, SUM, PatComm

    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    n = world
    shard = (args.total_bytes // 2 // n) // 8 * 8  # bf16 elements per rank shard
    params = torch.randn(shard, dtype=torch.bfloat16, device=dev)
    gathered = torch.empty(n * shard, dtype=torch.bfloat16, device=dev)
    grads = torch.randn(n * shard, dtype=torch.bfloat16, device=dev)
    gshard = torch.empty(shard, dtype=torch.bfloat16, device=dev)
    for cap_mib in [int(x) for x in args.caps.split(",")]:
        comm = PatComm.from_process_group(device=local, staging_bytes=cap_mib << 20)
        if args.windows:  # zero copy: direct all-gather into `gathered`, PULL reduce-scatter from `grads`
            for t in (params, gathered, grads, gshard):
                comm.register(t)
        plan_ag, plan_rs = comm.plan(0, shard, BFLOAT16), comm.plan(1, shard, BFLOAT16)

        from paper_2506_20252_b200 import group

        def step():
            if args.group:
                with group():
                    comm.all_gather_into_tensor(gathered, params)
                    comm.reduce_scatter_tensor(gshard, grads, SUM)
            else:
                comm.all_gather_into_tensor(gathered, params)
                comm.reduce_scatter_tensor(gshard, grads, SUM)

        for _ in range(3):
            step()
        torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.iters):
            step()
        b.record()
        torch.cuda.synchronize()
        ms = torch.tensor([a.elapsed_time(b) / args.iters], device=dev)
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        comm.raise_async_error()
        # the gathered tensor must be every rank's shard in rank order
        ok = torch.tensor([1.0], device=dev)
        ref = [torch.empty_like(params) for _ in range(n)]
        dist.all_gather(ref, params)
        if not torch.equal(torch.cat(ref), gathered):
            ok.zero_()
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        bytes_ = 2 * (n - 1) * shard * 2
        nccl_ms = None
        if args.nccl:
            def nstep():
                dist.all_gather_into_tensor(gathered, params)
                dist.reduce_scatter_tensor(gshard, grads)
            for _ in range(3):
                nstep()
            torch.cuda.synchronize()
            dist.barrier()
            a.record()
            for _ in range(args.iters):
                nstep()
            b.record()
            torch.cuda.synchronize()
            t = torch.tensor([a.elapsed_time(b) / args.iters], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            nccl_ms = float(t)
        if rank == 0:
            print(json.dumps({"config": "zero3", "n": n, "dtype": "bf16", "total_bytes": args.total_bytes,
                              "shard_bytes": shard * 2, "staging_cap_mib": cap_mib,
                              "pool_bytes_ag": plan_ag["pool_bytes"], "pool_bytes_rs": plan_rs["pool_bytes"],
                              "slice_bytes": plan_ag["slice_bytes"], "protocol": [plan_ag["protocol"], plan_rs["protocol"]],
                              "peak_intermediate_slots": plan_ag["peak_intermediate_slots"],
                              "ms_per_step": float(ms), "busbw_gbs": bytes_ / (float(ms) * 1e-3) / 1e9,
                              "allgather_matches_nccl": bool(ok.item()), "windows": args.windows, "grouped": args.group,
                              "staging_bytes_used": [plan_ag.get("staging_bytes_used"), plan_rs.get("staging_bytes_used")],
                              "nccl_ms_per_step": nccl_ms, "nccl_algo": os.environ.get("NCCL_ALGO")}), flush=True)
        comm.destroy()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
