"""Single-process multi-GPU sweep (patCommInitAll over every visible GPU, one rank per GPU):
the north-star process model, where all-gather runs zero-copy into the peers' recvbufs.

  python tools/sp_sweep.py --out gpurun_out/sp4.json
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/sp.json")
    ap.add_argument("--min-bytes", type=int, default=1 << 20)
    ap.add_argument("--max-bytes", type=int, default=1 << 30)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--direct", type=int, default=0)
    ap.add_argument("--protocol", type=int, default=0, help="0 auto, 1 LL, 2 SIMPLE, 3 PULL")
    ap.add_argument("--gpus", type=int, default=0, help="ranks = first N GPUs (default all)")
    ap.add_argument("--tag", default="")
    args = ap.parse_args()
    import torch

    from paper_2506_20252_b200 import FLOAT32, SUM, PatComm

    n = args.gpus or torch.cuda.device_count()
    comm = PatComm.init_all(n, list(range(n)), direct=args.direct, protocol=args.protocol)
    out = open(args.out, "a")
    C = args.min_bytes
    while C <= args.max_bytes:
        elems = C // 4
        for coll in ("ag", "rs"):
            if coll == "ag":
                s = [torch.ones(elems, device=f"cuda:{d}") for d in range(n)]
                r = [torch.empty(n * elems, device=f"cuda:{d}") for d in range(n)]
                fn = lambda: comm.all_gather(s, r, elems, FLOAT32)
            else:
                s = [torch.ones(n * elems, device=f"cuda:{d}") for d in range(n)]
                r = [torch.empty(elems, device=f"cuda:{d}") for d in range(n)]
                fn = lambda: comm.reduce_scatter(s, r, elems, FLOAT32, SUM)
            for _ in range(3):
                fn()
            for d in range(n):
                torch.cuda.synchronize(d)
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
            for d in range(n):
                with torch.cuda.device(d):
                    ev[d][0].record()
            for _ in range(args.iters):
                fn()
            for d in range(n):
                with torch.cuda.device(d):
                    ev[d][1].record()
            for d in range(n):
                torch.cuda.synchronize(d)
            us = max(a.elapsed_time(b) for a, b in ev) * 1e3 / args.iters
            rec = {"coll": coll, "impl": "pat-sp", "n": n, "dtype": "f32", "bytes_per_rank": C, "us": us,
                   "busbw_gbs": (n - 1) * C / (us * 1e-6) / 1e9, "plan": comm.plan(0 if coll == "ag" else 1, elems, FLOAT32),
                   "direct": args.direct, "protocol": args.protocol, "tag": args.tag}
            out.write(json.dumps(rec) + "\n")
            out.flush()
            del s, r
        C *= 2
    comm.raise_async_error()
    comm.destroy()


if __name__ == "__main__":
    main()
