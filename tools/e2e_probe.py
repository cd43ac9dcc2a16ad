"""Where the N=1 end-to-end step's time goes: the bench's e2e loop (pinned host buffers, one H2D and
one D2H stream, two device buffer sets, grouped AG + RS of 8 ranks on one GPU) with events around
every copy and every step. Prints per-step medians and the overlap.

    python tools/e2e_probe.py [--steps 20] [--sets 2]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2506_20252_b200 import FLOAT32, SUM, PatComm, group  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--sets", type=int, default=2)
    a = ap.parse_args()
    n, elems = 8, 1 << 18
    dev = torch.device("cuda:0")
    comm = PatComm.init_all(n, [0] * n)
    hb = {k: torch.empty(n * m * elems, dtype=torch.float32).pin_memory()
          for k, m in (("ag_send", 1), ("rs_send", n), ("ag_recv", n), ("rs_recv", 1))}
    for v in hb.values():
        v.uniform_()
    sets = [{k: torch.empty(n * m * elems, device=dev) for k, m in
             (("ag_send", 1), ("rs_send", n), ("ag_recv", n), ("rs_recv", 1))} for _ in range(a.sets)]
    main_s, s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    E = a.steps
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    marks = [{k: ev() for k in ("h0", "h1", "c0", "c1", "d0", "d1")} for _ in range(E)]
    t0, t1 = ev(), ev()
    S = a.sets

    def step_call(bs):
        v = {k: list(t.view(n, -1)) for k, t in bs.items()}
        with group():
            comm.all_gather(v["ag_send"], v["ag_recv"], elems, FLOAT32, streams=[main_s] * n)
            comm.reduce_scatter(v["rs_send"], v["rs_recv"], elems, FLOAT32, SUM, streams=[main_s] * n)

    for _ in range(2):
        step_call(sets[0])
    torch.cuda.synchronize()
    t0.record(main_s)
    s_in.wait_stream(main_s)
    s_out.wait_stream(main_s)
    for k in range(E):
        bs = sets[k % S]
        with torch.cuda.stream(s_in):
            if k >= S:
                s_in.wait_event(marks[k - S]["c1"])
            marks[k]["h0"].record(s_in)
            bs["ag_send"].copy_(hb["ag_send"], non_blocking=True)
            bs["rs_send"].copy_(hb["rs_send"], non_blocking=True)
            marks[k]["h1"].record(s_in)
        main_s.wait_event(marks[k]["h1"])
        if k >= S:
            main_s.wait_event(marks[k - S]["d1"])
        marks[k]["c0"].record(main_s)
        step_call(bs)
        marks[k]["c1"].record(main_s)
        with torch.cuda.stream(s_out):
            s_out.wait_event(marks[k]["c1"])
            marks[k]["d0"].record(s_out)
            hb["ag_recv"].copy_(bs["ag_recv"], non_blocking=True)
            hb["rs_recv"].copy_(bs["rs_recv"], non_blocking=True)
            marks[k]["d1"].record(s_out)
    main_s.wait_event(marks[E - 1]["d1"])
    t1.record(main_s)
    torch.cuda.synchronize()
    total = t0.elapsed_time(t1)
    h = [m["h0"].elapsed_time(m["h1"]) for m in marks]
    d = [m["d0"].elapsed_time(m["d1"]) for m in marks]
    c = [m["c0"].elapsed_time(m["c1"]) for m in marks]
    # gaps: H2D(k+1) start - H2D(k) end
    hg = [marks[k]["h1"].elapsed_time(marks[k + 1]["h0"]) for k in range(E - 1)]
    print(json.dumps({"sets": S, "ms_per_step": total / E, "h2d_ms_med": statistics.median(h),
                      "d2h_ms_med": statistics.median(d), "compute_ms_med": statistics.median(c),
                      "h2d_gap_ms_med": statistics.median(hg),
                      "h2d_gbs": (9 * n * elems * 4) / (statistics.median(h) * 1e-3) / 1e9,
                      "d2h_gbs": (9 * n * elems * 4) / (statistics.median(d) * 1e-3) / 1e9}))
    comm.destroy()


if __name__ == "__main__":
    main()
