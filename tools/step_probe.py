"""Why is a graph of K (all-gather, reduce-scatter) steps slower than K all-gathers plus K
reduce-scatters? torchrun, one process per GPU, 1 MiB fp32 per rank. Times graphs of K calls in
several orders, each replayed R times after a device barrier + spin, and prints per-replay
microseconds per call on every rank (JSON lines).

    torchrun --nproc-per-node 2 tools/step_probe.py [--k 20] [--reps 5]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2506_20252_b200 import FLOAT32, SUM, PatComm  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--k", type=int, default=20)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--elems", type=int, default=1 << 18)
    ap.add_argument("--sets", type=int, default=8)
    a = ap.parse_args()
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    n, e = world, a.elems
    comm = PatComm.from_process_group(device=local)
    st = torch.cuda.Stream(dev)
    sets = [{"as": torch.rand(e, device=dev), "ar": torch.empty(n * e, device=dev),
             "rs": torch.rand(n * e, device=dev), "rr": torch.empty(e, device=dev)} for _ in range(a.sets)]

    def ag(b):
        comm.all_gather([b["as"]], [b["ar"]], e, FLOAT32, streams=[st])

    def rs(b):
        comm.reduce_scatter([b["rs"]], [b["rr"]], e, FLOAT32, SUM, streams=[st])

    orders = {"ag": [ag], "rs": [rs], "ag_rs": [ag, rs], "ag_ag": [ag, ag], "rs_ag": [rs, ag], "rs_rs": [rs, rs]}
    with torch.cuda.stream(st):
        for _ in range(3):
            for b in sets:
                ag(b)
                rs(b)
    torch.cuda.synchronize()
    dist.barrier()
    out = {}
    for name, fns in orders.items():
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(st):
            g.capture_begin(capture_error_mode="relaxed")
            for k in range(a.k):
                for j, f in enumerate(fns):
                    f(sets[(k * len(fns) + j) % a.sets])
            g.capture_end()
        with torch.cuda.stream(st):
            g.replay()
        torch.cuda.synchronize()
        ts = []
        for _ in range(a.reps):
            dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(st):
                comm.barrier([st])
                torch.cuda._sleep(200_000)
                e0.record(st)
                g.replay()
                e1.record(st)
            torch.cuda.synchronize()
            ts.append(round(1e3 * e0.elapsed_time(e1) / (a.k * len(fns)), 2))
        out[name] = ts
        del g
    comm.raise_async_error()
    print(json.dumps({"rank": rank, "us_per_call": out, "k": a.k, "plan_ag": comm.plan(0, e, FLOAT32)["protocol_name"]}),
          flush=True)
    dist.barrier()
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
