"""Per-iteration fence cost of the SIMPLE sender from a PAT_TRACE capture (tools/trace_run.py):
for every CTA, the time from the last push of an iteration to its fence completing, and the
push time of the iteration itself."""
import sys

import numpy as np

for f in sys.argv[1:]:
    tr = np.load(f)["trace"]
    fence, push = [], []
    for c in range(tr.shape[0]):
        ev = [(int(tr[c, 0, e, 0]), int(tr[c, 0, e, 1]) >> 56) for e in range(tr.shape[2]) if tr[c, 0, e, 0]]
        last_push = None
        it_start = None
        for ns, code in ev:
            if code == 2 and it_start is None:  # credit (start of the first task of an iteration)
                it_start = ns
            if code == 3:
                last_push = ns
                if it_start is None:
                    it_start = ns
            if code == 4 and last_push is not None:
                fence.append(ns - last_push)
                if it_start is not None:
                    push.append(last_push - it_start)
                it_start = ns
                last_push = None
    fence, push = np.array(fence) / 1e3, np.array(push) / 1e3
    print(f"{f}: iterations {fence.size}: fence us median {np.median(fence):.2f} p90 {np.percentile(fence, 90):.2f}; "
          f"push us median {np.median(push):.2f}; fence share {fence.sum() / (fence.sum() + push.sum()):.2%}")
