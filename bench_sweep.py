"""Size sweeps of PAT all-gather / reduce-scatter against NCCL Ring (BASELINE configs 2-5).

Run under torchrun, one process per GPU (N >= 2), or plain (N = 1: logical ranks in local mode):

  torchrun --nproc-per-node 4 --master-addr 127.0.0.1 bench_sweep.py --out gpurun_out/sweep4.json

Every point: W warm-up calls, then K calls timed with CUDA events (graph mode: the median over
--trials replays of a graph of K calls, each trial the max over ranks; loop mode: one pass, the
max over ranks). Calls run back to back without an L2 flush (the nccl-tests convention); events
mode flushes L2 before every call from 1 MiB up.
Writes one JSON object per line: {"coll", "impl", "n", "dtype", "bytes_per_rank", "us", "busbw_gbs"}.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/sweep.json")
    ap.add_argument("--min-bytes", type=int, default=8)
    ap.add_argument("--max-bytes", type=int, default=1 << 30)
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--dtypes", default="f32,bf16")
    ap.add_argument("--colls", default="ag,rs")
    ap.add_argument("--ranks", type=int, default=8, help="logical ranks when run without torchrun")
    ap.add_argument("--no-nccl", action="store_true")
    ap.add_argument("--protocol", type=int, default=0)
    ap.add_argument("--algos", default="pat", help="pat,ring: schedules run on the PAT transport "
                    "(ring = ring_allgather / its mirror through the generic executor, impl 'pat-ring')")
    ap.add_argument("--windows", action="store_true",
                    help="torchrun: user buffers inside registered symmetric windows (zero copy)")
    ap.add_argument("--trials", type=int, default=5, help="graph mode: timed replays per point (median)")
    ap.add_argument("--mode", default="loop", choices=["loop", "events", "graph"],
                    help="loop: K back-to-back calls between two events (nccl-tests style); events: one "
                         "event pair per call (median); graph: K calls captured in a CUDA graph")
    args = ap.parse_args()

    import torch
    import torch.distributed as dist

    from paper_2506_20252_b200 import BFLOAT16, FLOAT32, SUM, PatComm
    from paper_2506_20252_b200 import schedule as S

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    cfg = {"protocol": args.protocol} if args.protocol else {}
    if world > 1:
        os.environ.setdefault("NCCL_ALGO", "Ring")
        dist.init_process_group("nccl", device_id=dev)
        n = world
        comm = PatComm.from_process_group(device=local, **cfg)
        L = 1
    else:
        n = args.ranks
        comm = PatComm.init_all(n, [local] * n, **cfg)
        L = n
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    win = None
    if args.windows and world > 1:  # one pair of windows for every size, buffers at offset 0
        wbytes = (n + 1) * args.max_bytes + 4096
        win = (torch.empty(wbytes, dtype=torch.uint8, device=dev), torch.empty(wbytes, dtype=torch.uint8, device=dev))
        comm.register(win[0])
        comm.register(win[1])
    scheds = {}
    for a in args.algos.split(","):
        if a == "ring":
            scheds["pat-ring"] = (S.ring_allgather(n), S.mirror_schedule(S.ring_allgather(n)))
        else:
            scheds["pat"] = (None, None)
    from paper_2506_20252_b200 import INT32
    dts = {"f32": (torch.float32, FLOAT32), "bf16": (torch.bfloat16, BFLOAT16), "i32": (torch.int32, INT32)}
    out = open(args.out, "w") if rank == 0 else None

    def timed(fn, big):
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        if args.mode == "events":
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(args.iters)]
            for a, b in evs:
                if big:
                    flush.zero_()
                a.record(stream)
                fn()
                b.record(stream)
            torch.cuda.synchronize(dev)
            ts = sorted(a.elapsed_time(b) for a, b in evs)
            us = ts[len(ts) // 2] * 1e3
        else:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if args.mode == "graph":
                g = torch.cuda.CUDAGraph()
                s2 = torch.cuda.Stream(dev)
                s2.wait_stream(stream)
                with torch.cuda.stream(s2):
                    with torch.cuda.graph(g, stream=s2):
                        for _ in range(args.iters):
                            fn()
                stream.wait_stream(s2)
                g.replay()
                torch.cuda.synchronize(dev)
                # several trials, each (barrier, one replay of K calls); per trial the max over ranks,
                # then the median over trials: one rank entering a replay late (host jitter after
                # the barrier) inflates one trial, not the point
                trials = []
                for _ in range(args.trials):
                    if world > 1:
                        dist.barrier()
                    a.record(stream)
                    g.replay()
                    b.record(stream)
                    torch.cuda.synchronize(dev)
                    trials.append(a.elapsed_time(b) * 1e3 / args.iters)
                t = torch.tensor(trials, dtype=torch.float64, device=dev)
                if world > 1:
                    dist.all_reduce(t, op=dist.ReduceOp.MAX)
                return float(t.median().item())
            else:
                a.record(stream)
                for _ in range(args.iters):
                    fn()
                b.record(stream)
            torch.cuda.synchronize(dev)
            us = a.elapsed_time(b) * 1e3 / args.iters
        med = torch.tensor([us], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(med, op=dist.ReduceOp.MAX)
        return float(med.item())

    sizes = []
    b = args.min_bytes
    while b <= args.max_bytes:
        sizes.append(b)
        b *= 2
    for dname in args.dtypes.split(","):
        tdt, pdt = dts[dname]
        es = torch.empty(0, dtype=tdt).element_size()
        for C in sizes:
            elems = max(1, C // es)
            need = (n + 1) * elems * es * L * 2
            if need > 40 * (1 << 30):
                break
            big = C >= (1 << 20)
            for coll in args.colls.split(","):
                if win is not None:
                    sn, rn = (elems, n * elems) if coll == "ag" else (n * elems, elems)
                    s = [win[0][:sn * es].view(tdt)]
                    r = [win[1][:rn * es].view(tdt)]
                    s[0].fill_(1)
                elif coll == "ag":
                    s = [torch.ones(elems, dtype=tdt, device=dev) for _ in range(L)]
                    r = [torch.empty(n * elems, dtype=tdt, device=dev) for _ in range(L)]
                else:
                    s = [torch.ones(n * elems, dtype=tdt, device=dev) for _ in range(L)]
                    r = [torch.empty(elems, dtype=tdt, device=dev) for _ in range(L)]
                for impl, (sag, srs) in scheds.items():
                    if coll == "ag":
                        fn = lambda sc=sag: comm.all_gather(s, r, elems, pdt, schedule=sc)
                    else:
                        fn = lambda sc=srs: comm.reduce_scatter(s, r, elems, pdt, SUM, schedule=sc)
                    us = timed(fn, big)
                    rec = {"coll": coll, "impl": impl + ("-win" if win is not None else ""), "n": n, "gpus": world,
                           "dtype": dname, "bytes_per_rank": elems * es, "us": us,
                           "busbw_gbs": (n - 1) * elems * es / (us * 1e-6) / 1e9,
                           "plan": comm.plan(0 if coll == "ag" else 1, elems, pdt) if impl == "pat" else None,
                           "forced": args.protocol}
                    if out:
                        out.write(json.dumps(rec) + "\n")
                        out.flush()
                if world > 1 and not args.no_nccl:
                    if coll == "ag":
                        nfn = lambda: dist.all_gather_into_tensor(r[0], s[0])
                    else:
                        nfn = lambda: dist.reduce_scatter_tensor(r[0], s[0])
                    us = timed(nfn, big)
                    rec = {"coll": coll, "impl": "nccl-" + os.environ.get("NCCL_ALGO", "auto"), "n": n,
                           "gpus": world, "dtype": dname, "bytes_per_rank": elems * es, "us": us,
                           "busbw_gbs": (n - 1) * elems * es / (us * 1e-6) / 1e9}
                    if out:
                        out.write(json.dumps(rec) + "\n")
                        out.flush()
                del s, r
        torch.cuda.empty_cache()
    comm.raise_async_error()
    comm.destroy()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
