"""n = 8 ranks as 8 processes (one rank per process, the torchrun path bench.py --gpus 8 takes) on
however many GPUs the box has: rank r on cuda:(r % ngpu), handles exchanged over gloo (NCCL refuses
two ranks on one GPU). Every protocol and a few sizes, bit-exact against the CPU oracle on every
rank, then the 1 MiB AG + RS step timed from a CUDA graph (informative only: ranks sharing a GPU
share its SMs and links).

    torchrun --nproc-per-node 8 --master-addr 127.0.0.1 tools/mp8_check.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("PAT_TIMEOUT_MS", "20000")

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle as O  # noqa: E402
from paper_2506_20252_b200 import FLOAT32, SUM, PatComm  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    ngpu = torch.cuda.device_count()
    dev = torch.device(f"cuda:{rank % ngpu}")
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")
    n = world
    fails = 0
    for proto in (0, 1, 5, 2):  # auto, LL, LL32, SIMPLE
        comm = PatComm.from_process_group(device=dev.index, protocol=proto)
        for dt in (O.FLOAT32, O.BFLOAT16, O.INT32):
            for elems in (1, 4099, 1 << 18):
                seed = 31 * elems + dt + proto
                p = O.random_payload(dt, n, elems, seed)
                es = p.itemsize
                s = torch.from_numpy(p[rank * elems:(rank + 1) * elems].copy().view(np.uint8)).to(dev)
                r = torch.zeros(n * elems * es, dtype=torch.uint8, device=dev)
                comm.all_gather([s], [r], elems, dt)
                torch.cuda.synchronize(dev)
                want, _ = O.run_allgather(O.pat_allgather(n, O.max_trees(n)), dt, p, elems)
                if r.cpu().numpy().tobytes() != want[rank].tobytes():
                    fails += 1
                    print(f"rank {rank} AG mismatch proto={proto} dt={dt} elems={elems}", flush=True)
                q = O.random_payload(dt, n * n, elems, seed + 1)
                s = torch.from_numpy(q[rank * n * elems:(rank + 1) * n * elems].copy().view(np.uint8)).to(dev)
                r = torch.zeros(elems * es, dtype=torch.uint8, device=dev)
                comm.reduce_scatter([s], [r], elems, dt, O.SUM)
                torch.cuda.synchronize(dev)
                want, _ = O.run_reduce_scatter(O.pat_reduce_scatter(n, O.max_trees(n)), dt, O.SUM, q, elems)
                if r.cpu().numpy().tobytes() != want[rank].tobytes():
                    fails += 1
                    print(f"rank {rank} RS mismatch proto={proto} dt={dt} elems={elems}", flush=True)
        comm.raise_async_error()
        comm.destroy()
    # grouped all-gather + reduce-scatter (the bench's step), both orders, LL32 and SIMPLE sizes
    from paper_2506_20252_b200 import group
    comm = PatComm.from_process_group(device=dev.index)
    for elems in (1 << 18, 1 << 21):
        for rs_first in (False, True):
            p = O.random_payload(O.FLOAT32, n, elems, elems + 3 + rs_first)
            q = O.random_payload(O.FLOAT32, n * n, elems, elems + 5 + rs_first)
            s = torch.from_numpy(p[rank * elems:(rank + 1) * elems].copy()).to(dev)
            r = torch.zeros(n * elems, device=dev)
            s2 = torch.from_numpy(q[rank * n * elems:(rank + 1) * n * elems].copy()).to(dev)
            r2 = torch.zeros(elems, device=dev)
            with group():
                if rs_first:
                    comm.reduce_scatter([s2], [r2], elems, O.FLOAT32, O.SUM)
                    comm.all_gather([s], [r], elems, O.FLOAT32)
                else:
                    comm.all_gather([s], [r], elems, O.FLOAT32)
                    comm.reduce_scatter([s2], [r2], elems, O.FLOAT32, O.SUM)
            torch.cuda.synchronize(dev)
            want, _ = O.run_allgather(O.pat_allgather(n, O.max_trees(n)), O.FLOAT32, p, elems)
            fails += r.cpu().numpy().tobytes() != want[rank].tobytes()
            want, _ = O.run_reduce_scatter(O.pat_reduce_scatter(n, O.max_trees(n)), O.FLOAT32, O.SUM, q, elems)
            fails += r2.cpu().numpy().tobytes() != want[rank].tobytes()
    comm.raise_async_error()
    comm.destroy()
    # the bench step, informative
    comm = PatComm.from_process_group(device=dev.index)
    e = 1 << 18
    a_s, a_r = torch.rand(e, device=dev), torch.empty(n * e, device=dev)
    r_s, r_r = torch.rand(n * e, device=dev), torch.empty(e, device=dev)
    st = torch.cuda.Stream(dev)
    with torch.cuda.stream(st):
        for _ in range(5):
            comm.all_gather([a_s], [a_r], e, FLOAT32)
            comm.reduce_scatter([r_s], [r_r], e, FLOAT32, SUM)
    torch.cuda.synchronize(dev)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(st):
        g.capture_begin(capture_error_mode="relaxed")
        for _ in range(20):
            comm.all_gather([a_s], [a_r], e, FLOAT32)
            comm.reduce_scatter([r_s], [r_r], e, FLOAT32, SUM)
        g.capture_end()
        g.replay()
    torch.cuda.synchronize(dev)
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        comm.barrier([st])
        e0.record(st)
        g.replay()
        e1.record(st)
    torch.cuda.synchronize(dev)
    us = torch.tensor([1e3 * e0.elapsed_time(e1) / 20])
    dist.all_reduce(us, op=dist.ReduceOp.MAX)
    comm.raise_async_error()
    t = torch.tensor([fails])
    dist.all_reduce(t)
    if rank == 0:
        print(json.dumps({"MP8_RESULT": "ok" if int(t.item()) == 0 else "FAIL", "fails": int(t.item()), "world": world,
                          "gpus": ngpu, "step_us_shared_gpus": float(us.item()),
                          "plan_ag": comm.plan(0, e, FLOAT32)["protocol_name"]}), flush=True)
    comm.destroy()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
