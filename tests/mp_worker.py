"""Worker for tests/test_gpu_multiprocess.py: one process per GPU (torchrun), inbox pools
mapped with CUDA IPC; every rank checks its own output bit-exact against the CPU oracle."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle as O  # noqa: E402
from paper_2506_20252_b200 import PatComm  # noqa: E402


def group_section(rank, n, dev):
    """patGroupStart/End across processes: one launch runs the all-gather and the reduce-scatter on
    disjoint channel halves; bit-exact, both orders, LL32 and SIMPLE sizes."""
    from paper_2506_20252_b200 import group
    fails = 0
    comm = PatComm.from_process_group(device=dev.index)
    for elems in (3000, 1 << 18, 1 << 22):
        for rs_first in (False, True):
            p = O.random_payload(O.FLOAT32, n, elems, elems + rs_first)
            q = O.random_payload(O.FLOAT32, n * n, elems, elems + 7)
            s = torch.from_numpy(p[rank * elems:(rank + 1) * elems].copy()).to(dev)
            r = torch.zeros(n * elems, dtype=torch.float32, device=dev)
            s2 = torch.from_numpy(q[rank * n * elems:(rank + 1) * n * elems].copy()).to(dev)
            r2 = torch.zeros(elems, dtype=torch.float32, device=dev)
            with group():
                if rs_first:
                    comm.reduce_scatter([s2], [r2], elems, O.FLOAT32, O.SUM)
                    comm.all_gather([s], [r], elems, O.FLOAT32)
                else:
                    comm.all_gather([s], [r], elems, O.FLOAT32)
                    comm.reduce_scatter([s2], [r2], elems, O.FLOAT32, O.SUM)
            torch.cuda.synchronize(dev)
            want, _ = O.run_allgather(O.pat_allgather(n, O.max_trees(n)), O.FLOAT32, p, elems)
            if r.cpu().numpy().tobytes() != want[rank].tobytes():
                fails += 1
                print(f"rank {rank} grouped AG mismatch elems={elems} rs_first={rs_first}", flush=True)
            want, _ = O.run_reduce_scatter(O.pat_reduce_scatter(n, O.max_trees(n)), O.FLOAT32, O.SUM, q, elems)
            if r2.cpu().numpy().tobytes() != want[rank].tobytes():
                fails += 1
                print(f"rank {rank} grouped RS mismatch elems={elems} rs_first={rs_first}", flush=True)
    comm.raise_async_error()
    comm.destroy()
    return fails


def windows_section(rank, n, dev):
    """Symmetric windows (patCommRegister*): zero-copy direct all-gather, PULL reduce-scatter and
    PULL all-gather across processes, bit-exact; then a rank-dependent offset must be refused."""
    fails = 0
    elems = (1 << 20) + 7
    pad = 4096  # buffers sit at byte offset `pad` inside their windows, equal on every rank
    win_s = torch.zeros(n * elems * 4 + 2 * pad, dtype=torch.uint8, device=dev)
    win_r = torch.zeros(n * elems * 4 + 2 * pad, dtype=torch.uint8, device=dev)
    for proto in (0, 2, 3):  # auto, SIMPLE (direct all-gather), PULL
        comm = PatComm.from_process_group(device=local_of(dev), protocol=proto)
        comm.register(win_s)
        comm.register(win_r)
        for dt in (O.FLOAT32, O.INT32):
            p = O.random_payload(dt, n, elems, 77 + proto + dt)
            mine = p[rank * elems:(rank + 1) * elems]
            s = win_s[pad:pad + elems * 4]
            s.copy_(torch.from_numpy(mine.copy().view(np.uint8)))
            r = win_r[pad:pad + n * elems * 4]
            comm.all_gather([s], [r], elems, dt)
            torch.cuda.synchronize(dev)
            want, _ = O.run_allgather(O.pat_allgather(n, O.max_trees(n)), dt, p, elems)
            if r.cpu().numpy().tobytes() != want[rank].tobytes():
                fails += 1
                print(f"rank {rank} windowed AG mismatch proto={proto} dt={dt}", flush=True)
            q = O.random_payload(dt, n * n, elems, 99 + proto + dt)
            s = win_s[pad:pad + n * elems * 4]
            s.copy_(torch.from_numpy(q[rank * n * elems:(rank + 1) * n * elems].copy().view(np.uint8)))
            r = win_r[pad:pad + elems * 4]
            comm.reduce_scatter([s], [r], elems, dt, O.SUM)
            torch.cuda.synchronize(dev)
            want, _ = O.run_reduce_scatter(O.pat_reduce_scatter(n, O.max_trees(n)), dt, O.SUM, q, elems)
            if r.cpu().numpy().tobytes() != want[rank].tobytes():
                fails += 1
                print(f"rank {rank} windowed RS mismatch proto={proto} dt={dt}", flush=True)
            # in place inside the window: the send slice is the rank's slot of the receive buffer
            # (all-gather) / the receive slice is the rank's block of the send buffer (reduce-scatter)
            r = win_r[pad:pad + n * elems * 4]
            r.zero_()
            r[rank * elems * 4:(rank + 1) * elems * 4].copy_(torch.from_numpy(mine.copy().view(np.uint8)))
            comm.all_gather([r[rank * elems * 4:(rank + 1) * elems * 4]], [r], elems, dt)
            torch.cuda.synchronize(dev)
            want, _ = O.run_allgather(O.pat_allgather(n, O.max_trees(n)), dt, p, elems)
            if comm.async_error() or r.cpu().numpy().tobytes() != want[rank].tobytes():
                fails += 1
                print(f"rank {rank} windowed in-place AG mismatch proto={proto} dt={dt}", flush=True)
            s = win_s[pad:pad + n * elems * 4]
            s.copy_(torch.from_numpy(q[rank * n * elems:(rank + 1) * n * elems].copy().view(np.uint8)))
            comm.reduce_scatter([s], [s[rank * elems * 4:(rank + 1) * elems * 4]], elems, dt, O.SUM)
            torch.cuda.synchronize(dev)
            want, _ = O.run_reduce_scatter(O.pat_reduce_scatter(n, O.max_trees(n)), dt, O.SUM, q, elems)
            if comm.async_error() or s[rank * elems * 4:(rank + 1) * elems * 4].cpu().numpy().tobytes() != want[rank].tobytes():
                fails += 1
                print(f"rank {rank} windowed in-place RS mismatch proto={proto} dt={dt}", flush=True)
        # a grouped pair on windowed buffers (zero-copy all-gather + reduce-scatter in one launch)
        from paper_2506_20252_b200 import group
        p = O.random_payload(O.FLOAT32, n, elems, 123 + proto)
        q = O.random_payload(O.FLOAT32, n * n, elems, 321 + proto)
        half = n * elems * 4 + pad  # AG in the first half of each window's use, RS after it
        ws = torch.zeros(2 * half + pad, dtype=torch.uint8, device=dev)
        wr = torch.zeros(2 * half + pad, dtype=torch.uint8, device=dev)
        comm.register(ws)
        comm.register(wr)
        ag_s = ws[pad:pad + elems * 4]
        ag_s.copy_(torch.from_numpy(p[rank * elems:(rank + 1) * elems].copy().view(np.uint8)))
        ag_r = wr[pad:pad + n * elems * 4]
        rs_s = ws[half + pad:half + pad + n * elems * 4]
        rs_s.copy_(torch.from_numpy(q[rank * n * elems:(rank + 1) * n * elems].copy().view(np.uint8)))
        rs_r = wr[half + pad:half + pad + elems * 4]
        with group():
            comm.all_gather([ag_s], [ag_r], elems, O.FLOAT32)
            comm.reduce_scatter([rs_s], [rs_r], elems, O.FLOAT32, O.SUM)
        torch.cuda.synchronize(dev)
        want, _ = O.run_allgather(O.pat_allgather(n, O.max_trees(n)), O.FLOAT32, p, elems)
        if ag_r.cpu().numpy().tobytes() != want[rank].tobytes():
            fails += 1
            print(f"rank {rank} windowed grouped AG mismatch proto={proto}", flush=True)
        want, _ = O.run_reduce_scatter(O.pat_reduce_scatter(n, O.max_trees(n)), O.FLOAT32, O.SUM, q, elems)
        if rs_r.cpu().numpy().tobytes() != want[rank].tobytes():
            fails += 1
            print(f"rank {rank} windowed grouped RS mismatch proto={proto}", flush=True)
        comm.raise_async_error()
        comm.deregister(wr)
        comm.deregister(ws)
        comm.deregister(win_r)
        comm.deregister(win_s)
        comm.destroy()
    # rank-dependent offsets: the entry check refuses the zero-copy call on the ranks that see it
    comm = PatComm.from_process_group(device=local_of(dev), protocol=2, timeout_ms=3000)
    comm.register(win_r)
    off = pad + 16 * rank
    s = torch.zeros(elems * 4, dtype=torch.uint8, device=dev)
    comm.all_gather([s], [win_r[off:off + n * elems * 4]], elems, O.FLOAT32)
    torch.cuda.synchronize(dev)
    if comm.async_error() == 0:
        fails += 1
        print(f"rank {rank} mismatched window offsets were not refused", flush=True)
    comm.destroy()
    return fails


def local_of(dev):
    return dev.index


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    n = world
    fails = 0
    for proto in (0, 1, 2):  # auto, LL, SIMPLE (PULL needs one process for all ranks)
        comm = PatComm.from_process_group(device=local, protocol=proto)
        for trees in O.valid_tree_counts(n):
            for elems in (1, 37, 4096, 65537, 1 << 20):
                for dt in (O.FLOAT32, O.BFLOAT16, O.INT32):
                    if proto and elems == 1 << 20 and dt != O.FLOAT32:
                        continue
                    seed = 1000 * trees + elems + dt
                    p = O.random_payload(dt, n, elems, seed)
                    mine = p[rank * elems:(rank + 1) * elems].copy()
                    npdt = mine.dtype
                    s = torch.from_numpy(mine.view(np.uint8)).to(dev)
                    r = torch.zeros(n * elems * mine.itemsize, dtype=torch.uint8, device=dev)
                    sched = None
                    if trees != O.max_trees(n):
                        from paper_2506_20252_b200 import schedule as S
                        sched = S.pat_allgather(n, trees)
                    comm.all_gather([s], [r], elems, dt, schedule=sched)
                    torch.cuda.synchronize(dev)
                    want, _ = O.run_allgather(O.pat_allgather(n, trees), dt, p, elems)
                    got = r.cpu().numpy().view(npdt)
                    if got.tobytes() != want[rank].tobytes():
                        fails += 1
                        print(f"rank {rank} AG mismatch proto={proto} T={trees} elems={elems} dt={dt}", flush=True)
                    q = O.random_payload(dt, n * n, elems, seed + 1)
                    s = torch.from_numpy(q[rank * n * elems:(rank + 1) * n * elems].copy().view(np.uint8)).to(dev)
                    r = torch.zeros(elems * mine.itemsize, dtype=torch.uint8, device=dev)
                    if sched is not None:
                        from paper_2506_20252_b200 import schedule as S
                        sched = S.pat_reduce_scatter(n, trees)
                    comm.reduce_scatter([s], [r], elems, dt, O.SUM, schedule=sched)
                    torch.cuda.synchronize(dev)
                    want, _ = O.run_reduce_scatter(O.pat_reduce_scatter(n, trees), dt, O.SUM, q, elems)
                    got = r.cpu().numpy().view(npdt)
                    if got.tobytes() != want[rank].tobytes():
                        fails += 1
                        print(f"rank {rank} RS mismatch proto={proto} T={trees} elems={elems} dt={dt}", flush=True)
        comm.raise_async_error()
        comm.destroy()
    # torch.distributed-shaped forms (ZeRO-3 callers): all-gather equals NCCL's bit for bit,
    # reduce-scatter equals the PAT-order oracle
    comm = PatComm.from_process_group(device=local)
    for elems in (4099, 3 << 20):
        x = torch.randn(elems, device=dev).to(torch.bfloat16)
        out, ref = torch.empty(n * elems, dtype=torch.bfloat16, device=dev), torch.empty(n * elems, dtype=torch.bfloat16, device=dev)
        comm.all_gather_into_tensor(out, x)
        dist.all_gather_into_tensor(ref, x)
        torch.cuda.synchronize(dev)
        if not torch.equal(out, ref):
            fails += 1
            print(f"rank {rank} all_gather_into_tensor differs from NCCL elems={elems}", flush=True)
        q = O.random_payload(O.BFLOAT16, n * n, elems, elems + 17)
        g = torch.from_numpy(q[rank * n * elems:(rank + 1) * n * elems].copy().view(np.int16)).to(dev).view(torch.bfloat16)
        shard = torch.empty(elems, dtype=torch.bfloat16, device=dev)
        comm.reduce_scatter_tensor(shard, g)
        torch.cuda.synchronize(dev)
        want, _ = O.run_reduce_scatter(O.pat_reduce_scatter(n, O.max_trees(n)), O.BFLOAT16, O.SUM, q, elems)
        if shard.view(torch.int16).cpu().numpy().view(np.uint16).tobytes() != want[rank].tobytes():
            fails += 1
            print(f"rank {rank} reduce_scatter_tensor differs from the oracle elems={elems}", flush=True)
    # in-place forms (FSDP): the input is the rank's slot of the output / the output is the rank's
    # block of the input
    for elems in (4099, 3 << 20):
        x = torch.randn(elems, device=dev)
        out, ref = torch.zeros(n * elems, device=dev), torch.empty(n * elems, device=dev)
        out[rank * elems:(rank + 1) * elems] = x
        comm.all_gather_into_tensor(out, out[rank * elems:(rank + 1) * elems])
        dist.all_gather_into_tensor(ref, x)
        torch.cuda.synchronize(dev)
        if not torch.equal(out, ref):
            fails += 1
            print(f"rank {rank} in-place all_gather_into_tensor differs from NCCL elems={elems}", flush=True)
        q = O.random_payload(O.FLOAT32, n * n, elems, elems + 29)
        g = torch.from_numpy(q[rank * n * elems:(rank + 1) * n * elems].copy()).to(dev)
        comm.reduce_scatter_tensor(g[rank * elems:(rank + 1) * elems], g)
        torch.cuda.synchronize(dev)
        want, _ = O.run_reduce_scatter(O.pat_reduce_scatter(n, O.max_trees(n)), O.FLOAT32, O.SUM, q, elems)
        if g[rank * elems:(rank + 1) * elems].cpu().numpy().tobytes() != want[rank].tobytes():
            fails += 1
            print(f"rank {rank} in-place reduce_scatter_tensor differs from the oracle elems={elems}", flush=True)
    comm.raise_async_error()
    comm.destroy()
    fails += group_section(rank, n, dev)
    fails += windows_section(rank, n, dev)
    t = torch.tensor([fails], device=dev)
    dist.all_reduce(t)
    if rank == 0:
        print(f"MP_RESULT fails={int(t.item())} world={world}", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
