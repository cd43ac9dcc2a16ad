"""Single-process latency sweep in graph mode: one process drives every rank (patCommInitAll), the
north-star process model, so rank counts above the GPU count run with ranks sharing GPUs
round-robin (n = 5..8 on a 4-GPU box: the co-located ranks of a device run in the same kernel).

Every call launches one kernel per device; K calls are captured into one CUDA graph per device
(concurrent relaxed-mode captures on each device's stream), the graphs are replayed together,
and a point is the median over trials of the max over devices of (replay time / K).

  python tools/sp_graph.py --ranks 5,6,7,8 --out gpurun_out/sp_graph.jsonl
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ranks", default="5,6,7,8")
    ap.add_argument("--min-bytes", type=int, default=8)
    ap.add_argument("--max-bytes", type=int, default=1 << 20)
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--trials", type=int, default=5)
    ap.add_argument("--out", default="gpurun_out/sp_graph.jsonl")
    args = ap.parse_args()
    import torch

    from paper_2506_20252_b200 import FLOAT32, SUM, PatComm

    ngpu = torch.cuda.device_count()
    out = open(args.out, "a")
    for n in [int(x) for x in args.ranks.split(",")]:
        devices = [r % ngpu for r in range(n)]
        devs = sorted(set(devices))
        comm = PatComm.init_all(n, devices)
        streams = {d: torch.cuda.Stream(d) for d in devs}
        C = args.min_bytes
        while C <= args.max_bytes:
            elems = max(1, C // 4)
            for coll in ("ag", "rs"):
                if coll == "ag":
                    s = [torch.ones(elems, device=f"cuda:{d}") for d in devices]
                    r = [torch.empty(n * elems, device=f"cuda:{d}") for d in devices]
                    fn = lambda: comm.all_gather(s, r, elems, FLOAT32, streams=[streams[d] for d in devices])  # noqa: E731
                else:
                    s = [torch.ones(n * elems, device=f"cuda:{d}") for d in devices]
                    r = [torch.empty(elems, device=f"cuda:{d}") for d in devices]
                    fn = lambda: comm.reduce_scatter(s, r, elems, FLOAT32, SUM,  # noqa: E731
                                                     streams=[streams[d] for d in devices])
                for _ in range(5):
                    fn()
                for d in devs:
                    torch.cuda.synchronize(d)
                graphs = {d: torch.cuda.CUDAGraph() for d in devs}
                for d in devs:
                    with torch.cuda.device(d):
                        torch.cuda.set_stream(streams[d])
                        graphs[d].capture_begin(capture_error_mode="relaxed")
                for _ in range(args.iters):
                    fn()
                for d in devs:
                    with torch.cuda.device(d):
                        graphs[d].capture_end()
                        torch.cuda.set_stream(torch.cuda.default_stream(d))
                for d in devs:
                    with torch.cuda.device(d), torch.cuda.stream(streams[d]):
                        graphs[d].replay()  # replays on the current stream
                for d in devs:
                    torch.cuda.synchronize(d)
                trials = []
                for _ in range(args.trials):
                    ev = {d: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for d in devs}
                    for d in devs:
                        with torch.cuda.device(d), torch.cuda.stream(streams[d]):
                            ev[d][0].record(streams[d])
                            graphs[d].replay()
                            ev[d][1].record(streams[d])
                    for d in devs:
                        torch.cuda.synchronize(d)
                    trials.append(max(ev[d][0].elapsed_time(ev[d][1]) for d in devs) * 1e3 / args.iters)
                us = statistics.median(trials)
                plan = comm.plan(0 if coll == "ag" else 1, elems, FLOAT32)
                rec = {"coll": coll, "impl": "pat-sp-graph", "n": n, "gpus": len(devs), "devices": devices,
                       "dtype": "f32", "bytes_per_rank": elems * 4, "us": us,
                       "busbw_gbs": (n - 1) * elems * 4 / (us * 1e-6) / 1e9, "plan": plan}
                out.write(json.dumps(rec) + "\n")
                out.flush()
                del graphs, s, r
            C *= 2
        comm.raise_async_error()
        comm.destroy()


if __name__ == "__main__":
    main()
