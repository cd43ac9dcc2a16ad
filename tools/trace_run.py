"""Device event trace of one transport call per rank (diagnostics).

  PAT_TRACE=64 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tools/trace_run.py --bytes 16777216 --coll ag

SIMPLE calls trace in the default build. LL / LL32 calls need a diagnostic build:
  bash tools/build_variant.sh tracepoll -DPAT_TRACE_POLL=1    # then PAT_LIB_VARIANT=tracepoll PAT_TRACE=8 ...

Writes gpurun_out/trace_<coll>_<bytes>_r<rank>.npz (ctas x 2 roles x entries x {ns, code}) and
prints, for rank 0, a timeline summary: per event type, the min / median / max time (us) from
the kernel's first event, over CTAs.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

EV = {1: "start", 2: "credit", 3: "pushed", 4: "fenced", 5: "arrived", 6: "delivered", 7: "done", 8: "end"}


def summarize(tr):
    import numpy as np

    t0 = None
    rows = {}
    for c in range(tr.shape[0]):
        for role in range(2):
            for e in range(tr.shape[2]):
                ns, code = int(tr[c, role, e, 0]), int(tr[c, role, e, 1])
                if ns == 0:
                    continue
                t0 = ns if t0 is None else min(t0, ns)
                ev, step, rnd = code >> 56, (code >> 40) & 0xFFFF, (code >> 32) & 0xFF
                rows.setdefault((role, EV.get(ev, ev), rnd), []).append((ns, step))
    out = []
    for (role, ev, rnd), v in sorted(rows.items(), key=lambda kv: min(x[0] for x in kv[1])):
        ts = np.array([x[0] - t0 for x in v]) / 1e3
        out.append(f"{'push' if role == 0 else 'recv'} {ev:9s} r{rnd} n={len(ts):5d}  min {ts.min():8.2f}  "
                   f"med {np.median(ts):8.2f}  max {ts.max():8.2f} us")
    return "\n".join(out)


def channel_timeline(tr, cta):
    """Per event of one CTA (both roles), time in us from the CTA's first event: the per-iteration
    picture of credit waits, pushes, fences and arrivals."""
    rows = []
    for role in range(2):
        for e in range(tr.shape[2]):
            ns, code = int(tr[cta, role, e, 0]), int(tr[cta, role, e, 1])
            if ns:
                rows.append((ns, "push" if role == 0 else "recv", EV.get(code >> 56, code >> 56),
                             (code >> 40) & 0xFFFF, (code >> 32) & 0xFF))
    if not rows:
        return ""
    t0 = min(r[0] for r in rows)
    return "\n".join(f"{(ns - t0) / 1e3:9.2f} {role} {ev:9s} step {st:5d} r{rd}" for ns, role, ev, st, rd in sorted(rows))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bytes", type=int, default=16 << 20)
    ap.add_argument("--coll", default="ag")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--staging-mib", type=int, default=0, help="patConfig staging_bytes cap")
    ap.add_argument("--protocol", type=int, default=0)
    ap.add_argument("--dtype", default="f32", choices=["f32", "bf16"])
    args = ap.parse_args()
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2506_20252_b200 import BFLOAT16, FLOAT32, SUM, PatComm

    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    comm = PatComm.from_process_group(device=local, staging_bytes=args.staging_mib << 20,
                                      protocol=args.protocol or None)
    tdt, FLOAT32 = (torch.float32, FLOAT32) if args.dtype == "f32" else (torch.bfloat16, BFLOAT16)
    n, elems = world, args.bytes // (4 if args.dtype == "f32" else 2)
    if args.coll == "ag":
        s, r = torch.ones(elems, device=dev, dtype=tdt), torch.empty(n * elems, device=dev, dtype=tdt)
        fn = lambda: comm.all_gather([s], [r], elems, FLOAT32)
    else:
        s, r = torch.ones(n * elems, device=dev, dtype=tdt), torch.empty(elems, device=dev, dtype=tdt)
        fn = lambda: comm.reduce_scatter([s], [r], elems, FLOAT32, SUM)
    for _ in range(args.warmup):
        fn()
    torch.cuda.synchronize(dev)
    dist.barrier()
    comm.barrier()  # device barrier: both GPUs start the traced call together, host skew excluded
    fn()
    torch.cuda.synchronize(dev)
    tr = comm.trace()
    os.makedirs("gpurun_out", exist_ok=True)
    np.savez_compressed(f"gpurun_out/trace_{args.coll}_{args.bytes}_r{rank}.npz", trace=tr,
                        plan=str(comm.plan(0 if args.coll == "ag" else 1, elems, FLOAT32)))
    if rank == 0:
        print(comm.plan(0 if args.coll == "ag" else 1, elems, FLOAT32))
        print(summarize(tr))
        print(channel_timeline(tr, 0))
    dist.barrier()
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
