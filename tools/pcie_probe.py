"""PCIe copy ceilings on this box for the N=1 e2e shape (72 MiB each way per step): H2D alone, D2H
alone, both at once on two streams (pinned host memory, events). Prints one JSON line."""
import json
import torch

n = 72 << 20
h_in = torch.empty(n // 4, dtype=torch.float32).pin_memory()
h_out = torch.empty(n // 4, dtype=torch.float32).pin_memory()
d_in = torch.empty(n // 4, device="cuda")
d_out = torch.empty(n // 4, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
K = 20


def timed(fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s1.wait_stream(torch.cuda.current_stream())
    s2.wait_stream(torch.cuda.current_stream())
    for _ in range(K):
        fn()
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


def both():
    h2d()
    d2h()


out = {}
for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    ms = timed(fn)
    out[name + "_gbs"] = (2 if name == "both" else 1) * n / (ms * 1e-3) / 1e9
print(json.dumps(out))
