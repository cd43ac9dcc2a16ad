"""Host cost of one eager collective call through the Python binding (N=1 bench shape: 8 ranks on
cuda:0, 1 MiB fp32, fused executor), split into its parts. Prints one JSON line.

    python tools/eager_probe.py [--calls 4000]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2506_20252_b200 import FLOAT32, SUM, PatComm  # noqa: E402
from paper_2506_20252_b200 import _lib  # noqa: E402


def per_call_us(fn, calls, sync_every=100):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(calls):
        fn()
        if (i + 1) % sync_every == 0:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    return 1e6 * (time.perf_counter() - t0) / calls


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--calls", type=int, default=4000)
    ap.add_argument("--ranks", type=int, default=8)
    ap.add_argument("--elems", type=int, default=256)
    a = ap.parse_args()
    n, e = a.ranks, a.elems
    comm = PatComm.init_all(n, [0] * n)
    s = torch.cuda.Stream()
    send = [torch.rand(e, device="cuda") for _ in range(n)]
    recv = [torch.empty(n * e, device="cuda") for _ in range(n)]
    rs_send = [torch.rand(n * e, device="cuda") for _ in range(n)]
    rs_recv = [torch.empty(e, device="cuda") for _ in range(n)]
    out = {"ranks": n, "elems": e, "fast_module": comm._fast is not None}
    with torch.cuda.stream(s):
        for _ in range(50):
            comm.all_gather(send, recv, e, FLOAT32)
        out["ag_api_us"] = per_call_us(lambda: comm.all_gather(send, recv, e, FLOAT32), a.calls)
        out["rs_api_us"] = per_call_us(lambda: comm.reduce_scatter(rs_send, rs_recv, e, FLOAT32, SUM), a.calls)
        F = comm._fast
        if F is not None:
            sp, rp, st = [x.data_ptr() for x in send], [x.data_ptr() for x in recv], [s.cuda_stream] * n
            h = comm._hv
            out["ag_fast_raw_us"] = per_call_us(lambda: F.all_gather(h, sp, rp, e, FLOAT32, st), a.calls)
        comm._fast = None  # the ctypes path
        out["ag_ctypes_us"] = per_call_us(lambda: comm.all_gather(send, recv, e, FLOAT32), a.calls)
        comm._fast = F
        ev = torch.cuda.Event(enable_timing=True)
        out["event_record_us"] = per_call_us(lambda: ev.record(s), a.calls)
        out["current_stream_us"] = per_call_us(lambda: torch.cuda.current_stream(0).cuda_stream, a.calls)
        raw = torch._C._cuda_getCurrentRawStream
        out["raw_stream_us"] = per_call_us(lambda: raw(0), a.calls)
        out["data_ptr_x8_us"] = per_call_us(lambda: [x.data_ptr() for x in send], a.calls)
        x = torch.empty(1, device="cuda")
        out["torch_fill_kernel_us"] = per_call_us(lambda: x.fill_(1.0), a.calls)
    comm.destroy()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
