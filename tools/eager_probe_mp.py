"""Host cost of eager calls with one rank per process (torchrun), 1 MiB fp32: per call host time of
the Python API, of the raw _patfast entry, and device time of K back-to-back calls (events).

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/eager_probe_mp.py
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2506_20252_b200 import FLOAT32, PatComm  # noqa: E402


def main():
    rank, local = int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    n = dist.get_world_size()
    comm = PatComm.from_process_group(device=local)
    e = 1 << 18
    s, r = torch.rand(e, device=dev), torch.empty(n * e, device=dev)
    st = torch.cuda.Stream(dev)
    out = {"rank": rank}
    K = 400
    with torch.cuda.stream(st):
        for _ in range(20):
            comm.all_gather([s], [r], e, FLOAT32, streams=[st])
        torch.cuda.synchronize(dev)
        dist.barrier()
        # host time per call (the GPU keeps up or queues; no sync inside)
        t0 = time.perf_counter()
        for _ in range(K):
            comm.all_gather([s], [r], e, FLOAT32, streams=[st])
        out["api_host_us"] = 1e6 * (time.perf_counter() - t0) / K
        torch.cuda.synchronize(dev)
        dist.barrier()
        F, h = comm._fast, comm._hv
        sp, rp, sh = s.data_ptr(), r.data_ptr(), st.cuda_stream
        t0 = time.perf_counter()
        for _ in range(K):
            F.all_gather(h, sp, rp, e, FLOAT32, sh)
        out["raw_host_us"] = 1e6 * (time.perf_counter() - t0) / K
        torch.cuda.synchronize(dev)
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        comm.barrier([st])
        torch.cuda._sleep(int(os.environ.get("PROBE_SPIN", "20000000")))  # queue the K calls behind a ~10 ms spin
        e0.record(st)
        for _ in range(K):
            F.all_gather(h, sp, rp, e, FLOAT32, sh)
        e1.record(st)
        torch.cuda.synchronize(dev)
        out["device_us_per_call_queued"] = 1e3 * e0.elapsed_time(e1) / K
        # the same K calls from a CUDA graph, same buffers and streams
        g = torch.cuda.CUDAGraph()
        g.capture_begin(capture_error_mode="relaxed")
        for _ in range(K):
            F.all_gather(h, sp, rp, e, FLOAT32, sh)
        g.capture_end()
        g.replay()
        torch.cuda.synchronize(dev)
        dist.barrier()
        comm.barrier([st])
        torch.cuda._sleep(int(os.environ.get("PROBE_SPIN", "20000000")))
        e0.record(st)
        g.replay()
        e1.record(st)
        torch.cuda.synchronize(dev)
        out["graph_us_per_call"] = 1e3 * e0.elapsed_time(e1) / K
    comm.raise_async_error()
    print(json.dumps(out), flush=True)
    dist.barrier()
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
