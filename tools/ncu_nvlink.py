"""NVLink counters of the transport kernel under ncu (diagnostics; achieved NVLink GB/s).

ncu profiles one kernel at a time and waits for it to finish, but a PAT kernel waits for its
peers' kernels. One process drives every GPU here (patCommInitAll), so profiling only the LAST
device's launches works: the other devices' kernels were launched (unprofiled, asynchronously)
just before and run alongside. Kernel replay would re-run the profiled kernel without its
peers, so the whole application is replayed instead:

  PAT_LAUNCH_THREADS=0 ncu --devices 1 --replay-mode application --clock-control none -k regex:pat_ \\
      --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum \\
      --csv --log-file gpurun_out/ncu_nvlink.csv python tools/ncu_nvlink.py --gpus 2

Each case runs W warm-up calls and one measured call; in the log the measured call is the
last pat_kernel launch of each case (cases in the order printed).
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--cases", default="ag:268435456,rs:268435456,ag:4194304,rs:4194304")
    args = ap.parse_args()
    import torch

    # device 0's launch must be issued before ncu holds the profiled one: one submitting thread
    os.environ.setdefault("PAT_LAUNCH_THREADS", "0")
    from paper_2506_20252_b200 import FLOAT32, SUM, PatComm

    n = args.gpus
    comm = PatComm.init_all(n, list(range(n)))
    for case in args.cases.split(","):
        coll, nbytes = case.split(":")
        elems = int(nbytes) // 4
        if coll == "grp":  # a grouped all-gather + reduce-scatter (one pat_group_kernel launch)
            from paper_2506_20252_b200 import group
            s = [torch.ones(elems, device=f"cuda:{d}") for d in range(n)]
            r = [torch.empty(n * elems, device=f"cuda:{d}") for d in range(n)]
            s2 = [torch.ones(n * elems, device=f"cuda:{d}") for d in range(n)]
            r2 = [torch.empty(elems, device=f"cuda:{d}") for d in range(n)]

            def fn():
                with group():
                    comm.all_gather(s, r, elems, FLOAT32)
                    comm.reduce_scatter(s2, r2, elems, FLOAT32, SUM)
            kind = 0
        elif coll == "ag":
            s = [torch.ones(elems, device=f"cuda:{d}") for d in range(n)]
            r = [torch.empty(n * elems, device=f"cuda:{d}") for d in range(n)]
            fn = lambda: comm.all_gather(s, r, elems, FLOAT32)  # noqa: E731
            kind = 0
        else:
            s = [torch.ones(n * elems, device=f"cuda:{d}") for d in range(n)]
            r = [torch.empty(elems, device=f"cuda:{d}") for d in range(n)]
            fn = lambda: comm.reduce_scatter(s, r, elems, FLOAT32, SUM)  # noqa: E731
            kind = 1
        for _ in range(args.warmup + 1):
            fn()
            for d in range(n):
                torch.cuda.synchronize(d)
        plan = comm.plan(kind, elems, FLOAT32)
        print(f"case {coll} {nbytes} B/rank n={n}: protocol {plan['protocol']} channels {plan['channels']} "
              f"iterations {plan['iterations']} launches/device {args.warmup + 1}", flush=True)
        del s, r
    comm.raise_async_error()
    comm.destroy()


if __name__ == "__main__":
    main()
