"""One process, every GPU: H2D + D2H of 5 MiB per GPU per step from pinned host buffers allocated
(a) under the copy's own device context, (b) all under device 0 — the one-process e2e shape."""
import json
import torch

n = torch.cuda.device_count()
nb = 5 << 20
out = {}
for mode in ("own_device", "device0"):
    hs, ds, ss = [], [], []
    for d in range(n):
        with torch.cuda.device(d if mode == "own_device" else 0):
            hs.append((torch.empty(nb // 4).pin_memory(), torch.empty(nb // 4).pin_memory()))
        ds.append((torch.empty(nb // 4, device=f"cuda:{d}"), torch.empty(nb // 4, device=f"cuda:{d}")))
        ss.append((torch.cuda.Stream(d), torch.cuda.Stream(d)))
    K = 50
    for rep in range(2):
        for d in range(n):
            torch.cuda.synchronize(d)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
        for d in range(n):
            with torch.cuda.device(d):
                ev[d][0].record(ss[d][0])
                ss[d][1].wait_stream(ss[d][0])
        for k in range(K):
            for d in range(n):
                with torch.cuda.device(d):
                    with torch.cuda.stream(ss[d][0]):
                        ds[d][0].copy_(hs[d][0], non_blocking=True)
                    with torch.cuda.stream(ss[d][1]):
                        hs[d][1].copy_(ds[d][1], non_blocking=True)
        for d in range(n):
            with torch.cuda.device(d):
                ss[d][0].wait_stream(ss[d][1])
                ev[d][1].record(ss[d][0])
        for d in range(n):
            torch.cuda.synchronize(d)
        ms = max(ev[d][0].elapsed_time(ev[d][1]) for d in range(n))
    out[mode + "_gbs_total"] = 2 * n * nb * K / (ms * 1e-3) / 1e9
print(json.dumps(out))
