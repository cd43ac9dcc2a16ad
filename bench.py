"""Benchmark of the PAT hot path: one step = one PAT all-gather + one PAT reduce-scatter(sum).

Workload (BASELINE.json configs[0]): 1 MiB fp32 per rank (262,144 elements), all-gather of
one chunk per rank and reduce-scatter of n chunks per rank into one.
  * N = 1 (plain `python bench.py`): n = 8 logical ranks on cuda:0, one cooperative kernel
    per collective ("local mode"; every rank's data in one GPU's HBM -> HBM roofline).
  * N > 1 (torchrun, one process per GPU): n = N ranks over NVLink, inbox pools mapped with
    CUDA IPC. NCCL's Ring all-gather / reduce-scatter is timed on the same buffers as a
    comparison (`nccl_ring`).

metric: aggregate bus bandwidth of the step = 2 * n * (n-1) * C bytes / step time (GB/s);
every rank receives (n-1)*C per collective (test_simulate.cpp:101-111). Per-collective
latencies are reported beside it.

`--impl reference` times the reference's own CPU executor (oracle/_ref, compiled from
/root/reference/proj/src) on the host cores on the same n and C (int64 all-gather + float64
reduce-scatter: equal bytes), rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CHUNK_BYTES = 1 << 20  # 1 MiB per rank
PEAKS_FALLBACK = {"hbm_gbs": 6650.0}
L2_BYTES = 126 * 1000 * 1000
NVLINK_MEASURED_GBS = 770.0  # peer copy per direction (B200_PROFILING.md)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="pat", choices=["pat", "reference"])
    ap.add_argument("--chunk-bytes", type=int, default=CHUNK_BYTES)
    ap.add_argument("--ranks", type=int, default=0, help="logical ranks at N=1 (default 8)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-nccl", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    return ap.parse_args()


def dist_env():
    if "WORLD_SIZE" in os.environ and int(os.environ["WORLD_SIZE"]) > 1:
        return int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ.get("LOCAL_RANK", 0))
    return 0, 1, 0


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return PEAKS_FALLBACK, "fallback"


# ------------------------------------------------------------------ reference CPU path

def reference_time(n: int, chunk_bytes: int, seconds: float, mode: int = 1, max_steps: int = 10000):
    """The reference executor (oracle/_ref) on the host: run_allgather(int64) +
    run_reduce_scatter(float64, FloatSum) with equal bytes per chunk. Returns
    (seconds per step, steps, threads)."""
    import ctypes

    import numpy as np

    import oracle as O

    R = O.ref()
    elems = chunk_bytes // 8
    ag = O.pat_allgather(n, O.max_trees(n))
    rs = O.pat_reduce_scatter(n, O.max_trees(n))
    pin = np.zeros(n * elems, np.int64)
    R.ref_random_payload(0, O.INT64, n, elems, 0, pin.ctypes.data)
    pout = np.zeros(n * n * elems, np.int64)
    qin = np.zeros(n * n * elems, np.float64)
    R.ref_random_payload(1, O.FLOAT64, n, elems, 0, qin.ctypes.data)
    qout = np.zeros(n * elems, np.float64)
    threads = os.cpu_count() or 1
    st = np.zeros(600, np.int64)

    def one():
        rc = R.ref_run_allgather(ag.ctypes.data_as(O.I32P), len(ag), O.INT64, elems, pin.ctypes.data,
                                 pout.ctypes.data, st.ctypes.data_as(O.I64P), mode, threads)
        rc |= R.ref_run_reduce_scatter(rs.ctypes.data_as(O.I32P), len(rs), O.FLOAT64, elems, qin.ctypes.data,
                                       qout.ctypes.data, st.ctypes.data_as(O.I64P), mode, threads)
        assert rc == 0

    one()  # warm-up
    steps, t0 = 0, time.perf_counter()
    while True:
        one()
        steps += 1
        el = time.perf_counter() - t0
        if el >= seconds or steps >= max_steps:
            break
    return el / steps, steps, threads if mode else 1


def dbg(msg: str) -> None:
    if os.environ.get("BENCH_DEBUG"):
        print(f"[bench {os.environ.get('RANK', '0')}] {msg}", file=sys.stderr, flush=True)


def busbw_gbs(n: int, chunk_bytes: int, seconds: float) -> float:
    return 2.0 * n * (n - 1) * chunk_bytes / seconds / 1e9


# ------------------------------------------------------------------ clocks during the timed region

class ClockSampler:
    """NVML sampling of SM clock + throttle reasons every ~5 ms on one GPU."""

    def __init__(self, device: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            pass

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if mask & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------ PAT arm

def run_pat(args, rank, world, local):
    import torch
    import torch.distributed as dist

    from paper_2506_20252_b200 import FLOAT32, SUM, PatComm

    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    C = args.chunk_bytes
    elems = C // 4
    if world > 1:
        os.environ.setdefault("NCCL_ALGO", "Ring")  # affects only the NCCL comparison below
        dist.init_process_group("nccl", device_id=dev)
        n = world
        comm = PatComm.from_process_group(device=local)
        ranks_here = [rank]
        placement = f"{n} ranks on {n} GPUs (1 process per GPU, CUDA IPC pools)"
    else:
        n = args.ranks or 8
        comm = PatComm.init_all(n, [local] * n)
        ranks_here = list(range(n))
        placement = f"{n} logical ranks on 1 GPU (fused single-device executor, local.cu)"
    L = len(ranks_here)
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    # Inputs larger than L2: the step's buffers are rotated over S sets whose total exceeds
    # twice the 126 MB L2, so every timed step starts cold.
    step_bytes = L * 2 * (n + 1) * C
    S = max(2, -(-(2 * L2_BYTES) // step_bytes) + 1)
    sets = []
    for _ in range(S):
        sets.append({
            "ag_send": [torch.rand(elems, device=dev, generator=g) for _ in range(L)],
            "ag_recv": [torch.empty(n * elems, device=dev) for _ in range(L)],
            "rs_send": [torch.rand(n * elems, device=dev, generator=g) for _ in range(L)],
            "rs_recv": [torch.empty(elems, device=dev) for _ in range(L)],
        })
    ag_send, ag_recv, rs_send, rs_recv = (sets[0][k] for k in ("ag_send", "ag_recv", "rs_send", "rs_recv"))
    stream = torch.cuda.current_stream(dev)

    def step(bs=None):
        bs = bs or sets[0]
        comm.all_gather(bs["ag_send"], bs["ag_recv"], elems, FLOAT32)
        comm.reduce_scatter(bs["rs_send"], bs["rs_recv"], elems, FLOAT32, SUM)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    dbg("warmup")
    for _ in range(args.warmup):
        for bs in sets:
            step(bs)
    barrier()
    comm.raise_async_error()
    dbg("capture")
    # The timed region replays ONE CUDA graph holding exactly K steps (step k = PAT all-gather +
    # PAT reduce-scatter on buffer set k % S), captured from the C-ABI calls: the launches are
    # the library's own kernels back to back, without Python/ctypes host gaps. Two more graphs
    # of K all-gathers and K reduce-scatters give the per-collective latencies.
    K = args.steps
    G = min(K, 1000)  # steps per graph; the timed region replays it K // G times (+ a remainder graph)

    def capture(kinds, count):
        gph = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream(dev)
        cap.wait_stream(stream)
        with torch.cuda.stream(cap):
            with torch.cuda.graph(gph, stream=cap):
                for k in range(count):
                    bs = sets[k % S]
                    if "ag" in kinds:
                        comm.all_gather(bs["ag_send"], bs["ag_recv"], elems, FLOAT32)
                    if "rs" in kinds:
                        comm.reduce_scatter(bs["rs_send"], bs["rs_recv"], elems, FLOAT32, SUM)
        stream.wait_stream(cap)
        return gph

    rem = K % G
    graphs = {kinds: (capture(kinds, G), capture(kinds, rem) if rem else None)
              for kinds in (("ag", "rs"), ("ag",), ("rs",))}
    dbg("replay-warm")
    for full, part in graphs.values():
        full.replay()
        if part is not None:
            part.replay()
    barrier()
    dbg("timed")

    def timed_replay(kinds):
        full, part = graphs[kinds]
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        a.record(stream)
        for _ in range(K // G):  # exactly K steps: K // G replays of G steps + the remainder
            full.replay()
        if part is not None:
            part.replay()
        b.record(stream)
        barrier()
        return a.elapsed_time(b)

    with ClockSampler(local) as clocks:
        step_ms = timed_replay(("ag", "rs"))
        ag_ms, rs_ms = timed_replay(("ag",)), timed_replay(("rs",))
    comm.raise_async_error()
    tot = torch.tensor([step_ms, ag_ms, rs_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    tot_ms, ag_ms, rs_ms = (float(x) for x in tot.tolist())
    ms_per_step = tot_ms / K
    value = busbw_gbs(n, C, ms_per_step / 1e3)

    # ---- the same steps launched eagerly through the C ABI (apples-to-apples with NCCL eager)
    KE = min(K, 100)
    eev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(KE)]
    barrier()
    for k in range(KE):
        bs = sets[k % S]
        eev[k][0].record(stream)
        comm.all_gather(bs["ag_send"], bs["ag_recv"], elems, FLOAT32)
        eev[k][1].record(stream)
        comm.reduce_scatter(bs["rs_send"], bs["rs_recv"], elems, FLOAT32, SUM)
        eev[k][2].record(stream)
    barrier()
    et = torch.tensor([sum(e[0].elapsed_time(e[1]) for e in eev), sum(e[1].elapsed_time(e[2]) for e in eev)],
                      dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
    eager_us = {"all_gather": 1e3 * float(et[0]) / KE, "reduce_scatter": 1e3 * float(et[1]) / KE}

    dbg("e2e")
    # ---- e2e through the C ABI with host buffers (pinned), H2D + D2H inside the timed region
    h_ag_send = [torch.empty(elems, dtype=torch.float32).pin_memory() for _ in range(L)]
    h_rs_send = [torch.empty(n * elems, dtype=torch.float32).pin_memory() for _ in range(L)]
    h_ag_recv = [torch.empty(n * elems, dtype=torch.float32).pin_memory() for _ in range(L)]
    h_rs_recv = [torch.empty(elems, dtype=torch.float32).pin_memory() for _ in range(L)]
    for i in range(L):
        h_ag_send[i].copy_(ag_send[i].cpu())
        h_rs_send[i].copy_(rs_send[i].cpu())
    # Double-buffered: step k's inputs go up on a copy stream into device set k % 2 while step
    # k-1 runs, and step k-1's results come down on another copy stream (PCIe is full duplex, so
    # the two directions overlap); every step still copies all of its inputs in and its results
    # out inside the timed region.
    E = max(3, min(K, 20))
    dsets = [sets[j % len(sets)] for j in range(2)]
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    ev = lambda: torch.cuda.Event()  # noqa: E731
    h2d_done, comp_done, d2h_done = [ev() for _ in range(E)], [ev() for _ in range(E)], [ev() for _ in range(E)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record(stream)
    s_in.wait_stream(stream)
    s_out.wait_stream(stream)
    for k in range(E):
        bs = dsets[k % 2]
        with torch.cuda.stream(s_in):
            if k >= 2:
                s_in.wait_event(comp_done[k - 2])  # set k % 2's inputs are free
            for i in range(L):
                bs["ag_send"][i].copy_(h_ag_send[i], non_blocking=True)
                bs["rs_send"][i].copy_(h_rs_send[i], non_blocking=True)
            h2d_done[k].record(s_in)
        stream.wait_event(h2d_done[k])
        if k >= 2:
            stream.wait_event(d2h_done[k - 2])  # set k % 2's outputs were read back
        step(bs)
        comp_done[k].record(stream)
        with torch.cuda.stream(s_out):
            s_out.wait_event(comp_done[k])
            for i in range(L):
                h_ag_recv[i].copy_(bs["ag_recv"][i], non_blocking=True)
                h_rs_recv[i].copy_(bs["rs_recv"][i], non_blocking=True)
            d2h_done[k].record(s_out)
    stream.wait_event(d2h_done[E - 1])
    stream.wait_event(h2d_done[E - 1])
    e1.record(stream)
    barrier()
    e2e_ms = torch.tensor([e0.elapsed_time(e1) / E], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_ms = float(e2e_ms.item())
    h2d = L * (elems + n * elems) * 4
    d2h = L * (n * elems + elems) * 4

    # ---- NCCL Ring comparison (N > 1)
    nccl = None
    dbg("nccl")
    if world > 1 and not args.no_nccl:
        for _ in range(args.warmup):
            for bs in sets:
                dist.all_gather_into_tensor(bs["ag_recv"][0], bs["ag_send"][0])
                dist.reduce_scatter_tensor(bs["rs_recv"][0], bs["rs_send"][0])
        barrier()
        # same timing method as the PAT arm: graph replay when NCCL captures, else eager
        ngraphs, mode = [], "graph"
        dbg("nccl-capture")
        try:
            if not os.environ.get("BENCH_NCCL_GRAPH"):  # capturing many NCCL graphs hung on 2.28.9
                raise RuntimeError("eager")
            cap2 = torch.cuda.Stream(dev)
            cap2.wait_stream(stream)
            with torch.cuda.stream(cap2):
                for bs in sets:
                    ga, gr = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
                    with torch.cuda.graph(ga, stream=cap2):
                        dist.all_gather_into_tensor(bs["ag_recv"][0], bs["ag_send"][0])
                    with torch.cuda.graph(gr, stream=cap2):
                        dist.reduce_scatter_tensor(bs["rs_recv"][0], bs["rs_send"][0])
                    ngraphs.append((ga, gr))
            stream.wait_stream(cap2)
            for ga, gr in ngraphs:
                ga.replay()
                gr.replay()
        except Exception:
            mode, ngraphs = "eager", []
        barrier()
        KN = min(K, 1000)
        nev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(KN)]
        for k in range(KN):
            bs = sets[k % S]
            nev[k][0].record(stream)
            if ngraphs:
                ngraphs[k % S][0].replay()
            else:
                dist.all_gather_into_tensor(bs["ag_recv"][0], bs["ag_send"][0])
            nev[k][1].record(stream)
            if ngraphs:
                ngraphs[k % S][1].replay()
            else:
                dist.reduce_scatter_tensor(bs["rs_recv"][0], bs["rs_send"][0])
            nev[k][2].record(stream)
        barrier()
        nt = torch.tensor([sum(e[0].elapsed_time(e[2]) for e in nev), sum(e[0].elapsed_time(e[1]) for e in nev),
                           sum(e[1].elapsed_time(e[2]) for e in nev)], dtype=torch.float64, device=dev)
        dist.all_reduce(nt, op=dist.ReduceOp.MAX)
        nt = nt.tolist()
        nccl = {"algo": os.environ.get("NCCL_ALGO"), "ms_per_step": nt[0] / KN,
                "busbw_gbs": busbw_gbs(n, C, nt[0] / KN / 1e3),
                "ag_us": 1e3 * nt[1] / KN, "rs_us": 1e3 * nt[2] / KN,
                "nccl_version": ".".join(str(x) for x in torch.cuda.nccl.version()), "timing": mode}

    # ---- roofline of the dominant kernel
    peaks, peak_src = load_peaks()
    dom = "reduce_scatter" if rs_ms >= ag_ms else "all_gather"
    dom_us = 1e3 * max(ag_ms, rs_ms) / K
    if world == 1:
        algo_bytes = (n * n + n) * C  # local mode: read n*C + write n^2*C (AG) / read n^2*C + write n*C (RS)
        peak = float(peaks.get("hbm_gbs", PEAKS_FALLBACK["hbm_gbs"]))
        roof = {"bound": "hbm", "kernel": ("local_rs_kernel" if dom == "reduce_scatter" else "local_ag_tma_kernel"), "unit": "GB/s",
                "algorithmic_bytes_per_launch": algo_bytes, "peak_source": f"{peak_src} MEASURED_PEAKS.json hbm_gbs"}
    else:
        algo_bytes = (n - 1) * C  # per rank, received over NVLink
        peak = NVLINK_MEASURED_GBS
        roof = {"bound": "nvlink", "kernel": f"pat_kernel ({dom})", "unit": "GB/s",
                "algorithmic_bytes_per_launch": algo_bytes,
                "peak_source": "measured peer copy 770 GB/s per direction (B200_PROFILING.md)"}
    achieved = algo_bytes / (dom_us * 1e-6) / 1e9
    roof.update({"achieved": achieved, "peak": peak, "frac": achieved / peak, "traffic": None,
                 "launch_us": dom_us})
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            tr = json.load(open(tpath))
            key = f"{'local' if world == 1 else 'nvlink'}_n{n}_{dom}"
            if key in tr:
                roof["traffic"] = tr[key]["dram_bytes_per_launch"]
                roof["traffic_source"] = tr[key].get("source")
                if "nvlink_tx_bytes_per_launch" in tr[key]:  # NVLink egress of the same ncu launch
                    roof["nvlink_tx_bytes"] = tr[key]["nvlink_tx_bytes_per_launch"]
                    roof["nvlink_tx_user_bytes"] = tr[key]["nvlink_tx_user_bytes_per_launch"]
        except Exception:
            pass

    # small messages are latency-bound: compare with the PAT step floor — the zero-byte time of
    # R = ceil(log2 n) polling rounds (LL, the lowest fixed cost of the cost-model fit,
    # profiles/r01f_costmodel_fit.json) plus the payload on the wire with LL32's one flag word
    # per 28 bytes, at the measured two-way SM-push ceiling (profiles/r01_bidir_probe_g4.txt)
    lat_floor = None
    if world > 1:
        plan = comm.plan(0, elems, FLOAT32)
        R = plan["rounds"]
        zero_us = 3.41 + 1.40 * R
        wire_us = (32.0 / 28.0) * (n - 1) * C / (704.0 * 1e3)
        lat_floor = {"rounds": R, "protocol": plan["protocol"], "zero_byte_us": zero_us,
                     "wire_us_at_704gbs": wire_us, "floor_us": zero_us + wire_us, "achieved_us": 1e3 * ag_ms / K,
                     "frac": (zero_us + wire_us) / (1e3 * ag_ms / K),
                     "source": "profiles/r01f_costmodel_fit.json (LL a, b), profiles/r01_bidir_probe_g4.txt"}

    clk = clocks.summary()
    if world > 1:
        allc = [None] * world
        dist.all_gather_object(allc, clk)
        clk = {"sm_mhz": statistics.median([c["sm_mhz"] for c in allc if c["sm_mhz"]] or [0]),
               "sm_max_mhz": allc[0]["sm_max_mhz"], "reasons": sorted({r for c in allc for r in c["reasons"]}),
               "samples": sum(c["samples"] for c in allc)}

    plan_ag = comm.plan(0, elems, FLOAT32)
    plan_rs = comm.plan(1, elems, FLOAT32)
    out = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            try:
                sec, steps, thr = reference_time(n, C, args.cpu_seconds)
                cpu = {"value": busbw_gbs(n, C, sec), "unit": "GB/s", "cores": thr, "kind": "reference",
                       "ms_per_step": sec * 1e3,
                       "sample": f"{steps} steps of the reference executor (oracle/_ref = /root/reference/proj/src "
                                 f"compiled), n={n}, {C} B/rank, run_allgather(int64)+run_reduce_scatter(f64), "
                                 f"ExecMode::Parallel x{thr} threads, {args.cpu_seconds:.0f} s budget"}
            except Exception as e:  # the reference library must be built in-tree
                cpu = {"value": None, "unit": "GB/s", "cores": 0, "kind": "reference", "sample": f"unavailable: {e}"}
        out = {
            "metric": "PAT all-gather + reduce-scatter(sum) aggregate bus bandwidth, 1 MiB fp32 per rank",
            "value": value, "unit": "GB/s", "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (torch.rand on device)",
            "config": {"workload": "BASELINE configs[0]: PAT AG + RS(sum), 1 MiB fp32 per rank",
                       "nranks": n, "placement": placement, "chunk_bytes": C, "trees": plan_ag["trees"],
                       "rounds": plan_ag["rounds"], "l2": f"inputs larger than L2: {S} rotating buffer sets, {S * step_bytes / 2**20:.0f} MiB total",
                       "timing": "CUDA events around CUDA-graph replays of exactly K steps (captured C-ABI calls)",
                       "plan_allgather": plan_ag, "plan_reduce_scatter": plan_rs},
            "latency_us": {"all_gather": 1e3 * ag_ms / K, "reduce_scatter": 1e3 * rs_ms / K,
                           "timing": "graph of K back-to-back calls per collective"},
            "latency_us_eager": dict(eager_us, timing="eager C-ABI calls, CUDA events per call"),
            "e2e": {"value": busbw_gbs(n, C, e2e_ms / 1e3), "unit": "GB/s", "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "path": "pinned host -> device copies, patAllGather + patReduceScatter (C ABI), device -> host; double-buffered: step k+1 uploads while step k downloads (PCIe full duplex)"},
            "gpu_launches": 2 * K,
            "roofline": roof,
            "latency_floor": lat_floor,
            "cpu_baseline": cpu,
            "clocks": clk,
        }
        if nccl:
            out["nccl_ring"] = nccl
    comm.destroy()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return out


def run_reference(args, rank, world):
    if rank != 0:
        return None
    n = world if world > 1 else (args.ranks or 8)
    C = args.chunk_bytes
    # W warm-up steps (at most 3: each is the whole workload, ~90 ms), then exactly K timed steps
    # unless K steps would exceed ~2 minutes of host time: then as many as fit, reported in
    # "steps" and in the sample description
    for _ in range(min(args.warmup, 3)):
        reference_time(n, C, 0.0, max_steps=1)
    est, _, _ = reference_time(n, C, 0.0, max_steps=1)
    timed = max(1, min(args.steps, int(120.0 / max(est, 1e-6))))
    sec, steps, thr = reference_time(n, C, 1e9, max_steps=timed)
    budget = sec * steps
    value = busbw_gbs(n, C, sec)
    return {"impl": "reference", "metric": "PAT all-gather + reduce-scatter(sum) aggregate bus bandwidth, 1 MiB fp32 per rank",
            "value": value, "unit": "GB/s", "n_gpus": world, "steps": steps, "warmup": args.warmup,
            "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "int64 AG + f64 RS (equal bytes)", "data": "synthetic (reference mt19937_64 payloads)",
            "config": {"workload": "BASELINE configs[0]: PAT AG + RS(sum), 1 MiB per rank", "nranks": n,
                       "chunk_bytes": C, "placement": "in-process ranks on host cores"},
            "cpu_baseline": {"value": value, "unit": "GB/s", "cores": thr, "kind": "reference",
                             "sample": f"{steps} timed steps (of --steps {args.steps}) of the whole workload, "
                                       f"ExecMode::Parallel x{thr} threads, {budget:.1f} s"},
            "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    args = parse()
    # one JSON line on stdout: everything else (NCCL banners, warnings) goes to stderr
    real_stdout = os.dup(1)
    os.dup2(2, 1)
    sys.stdout = os.fdopen(os.dup(2), "w")
    rank, world, local = dist_env()
    if args.impl == "reference":
        out = run_reference(args, rank, world)
    else:
        out = run_pat(args, rank, world, local)
    if rank == 0 and out is not None:
        with os.fdopen(real_stdout, "w") as f:
            f.write(json.dumps(out) + "\n")


if __name__ == "__main__":
    main()
