"""Single-process latency sweep with n ranks spread round-robin over the visible GPUs, timed as
CUDA graphs (one multi-device graph per size: fork from device 0's stream to every device's
stream, K back-to-back collectives, join). This is how n = 5..8 ranks run on a 4-GPU box: two
ranks share a GPU and one cooperative kernel per GPU drives both, so half of each rank's peers
are reached through HBM instead of NVLink — a lower bound on the 8-GPU latency, not a
measurement of it. NCCL cannot place two ranks on one GPU, so there is no NCCL column.

  python tools/sp_latency.py --ranks 8 --out gpurun_out/sp_lat_n8.jsonl
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ranks", type=int, required=True)
    ap.add_argument("--min-bytes", type=int, default=8)
    ap.add_argument("--max-bytes", type=int, default=4 << 20)
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--out", required=True)
    args = ap.parse_args()
    import torch

    from paper_2506_20252_b200 import FLOAT32, SUM, PatComm

    G = torch.cuda.device_count()
    n = args.ranks
    devs = [r % G for r in range(n)]
    used = sorted(set(devs))
    comm = PatComm.init_all(n, devs)
    streams = {d: torch.cuda.Stream(device=d) for d in used}
    out = open(args.out, "a")
    C = args.min_bytes
    while C <= args.max_bytes:
        elems = max(1, C // 4)
        for coll in ("ag", "rs"):
            if coll == "ag":
                s = [torch.ones(elems, device=f"cuda:{d}") for d in devs]
                r = [torch.empty(n * elems, device=f"cuda:{d}") for d in devs]
            else:
                s = [torch.ones(n * elems, device=f"cuda:{d}") for d in devs]
                r = [torch.empty(elems, device=f"cuda:{d}") for d in devs]
            st = [streams[d] for d in devs]

            def call():
                if coll == "ag":
                    comm.all_gather(s, r, elems, FLOAT32, streams=st)
                else:
                    comm.reduce_scatter(s, r, elems, FLOAT32, SUM, streams=st)

            for _ in range(3):
                call()
            for d in used:
                torch.cuda.synchronize(d)
            s0 = streams[used[0]]
            g = torch.cuda.CUDAGraph()
            with torch.cuda.device(used[0]):
                with torch.cuda.graph(g, stream=s0):
                    fork = torch.cuda.Event()
                    fork.record(s0)
                    for d in used[1:]:
                        streams[d].wait_event(fork)
                    for _ in range(args.iters):
                        call()
                    for d in used[1:]:
                        j = torch.cuda.Event()
                        j.record(streams[d])
                        s0.wait_event(j)
            g.replay()
            for d in used:
                torch.cuda.synchronize(d)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.device(used[0]):
                a.record(s0)
                g.replay()
                b.record(s0)
            for d in used:
                torch.cuda.synchronize(d)
            us = a.elapsed_time(b) * 1e3 / args.iters
            rec = {"coll": coll, "impl": "pat-sp-graph", "n": n, "gpus": len(used), "dtype": "f32",
                   "bytes_per_rank": elems * 4, "us": us, "busbw_gbs": (n - 1) * elems * 4 / (us * 1e-6) / 1e9,
                   "plan": comm.plan(0 if coll == "ag" else 1, elems, FLOAT32), "placement": devs}
            out.write(json.dumps(rec) + "\n")
            out.flush()
            del g, s, r
        C *= 8 if C < 65536 else 2
    comm.raise_async_error()
    comm.destroy()


if __name__ == "__main__":
    main()
