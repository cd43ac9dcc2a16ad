"""Benchmark of the PAT hot path: one step = one PAT all-gather + one PAT reduce-scatter(sum).

Workload (BASELINE.json configs[0]): 1 MiB fp32 per rank (262,144 elements), all-gather of
one chunk per rank and reduce-scatter of n chunks per rank into one.

Placement, chosen from how the script is launched:
  * N = 1 (`python bench.py`): n = 8 logical ranks on cuda:0 (the reference's in-process ranks,
    BASELINE configs[0] exactly); the fused single-device executor (local.cu) runs it — every
    rank's data in one GPU's HBM, so the HBM roofline applies. The same n = 8 call through the
    PAT transport kernel (per-round messages and flags, `fused = -1`) is timed beside it
    (`transport_local`).
  * N > 1 under torchrun (the driver's form; WORLD_SIZE = N): n = N ranks, one process per
    GPU, inbox pools mapped with CUDA IPC; NCCL's Ring all-gather / reduce-scatter is timed on
    the same buffers the same way (CUDA graphs) as the comparison (`nccl_ring`).
  * N > 1 without torchrun (`python bench.py --gpus N [--ranks M]`): ONE process drives all N
    GPUs (patCommInitAll, the north-star process model); M ranks (default N) placed round-robin,
    e.g. `--gpus 4 --ranks 8` puts the n = 8 workload on devices [0,1,2,3,0,1,2,3].
  A line whose n_gpus differs from --gpus is never printed: a mismatch exits with status 2.

metric: aggregate bus bandwidth of the step = 2 * n * (n-1) * C bytes / step time (GB/s);
every rank receives (n-1)*C per collective (test_simulate.cpp:101-111). Per-collective
latencies are reported beside it.

`--impl reference` times the reference's own CPU executor (oracle/_ref, compiled from
/root/reference/proj/src) on the host cores on the same n and C (int64 all-gather + float64
reduce-scatter: equal bytes; the reference supports only those), rank 0 only.
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
NVLINK_PEER_COPY_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md)
NVLINK_NOMINAL_GBS = 900.0    # NVLink 5, 18 links, per direction per GPU
NVLINK_SM_PUSH_GBS = 704.0    # SM stores into peers, every GPU sending (profiles/r01_bidir_probe_g4.txt)


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="pat", choices=["pat", "reference"])
    ap.add_argument("--chunk-bytes", type=int, default=CHUNK_BYTES)
    ap.add_argument("--ranks", type=int, default=0,
                    help="ranks without torchrun (default: 8 at --gpus 1, else --gpus), placed round-robin")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-nccl", action="store_true")
    ap.add_argument("--nccl-graph", action="store_true", help="time NCCL Ring from CUDA graphs (hangs on some boxes)")
    ap.add_argument("--no-group", action="store_true", help="issue a step's all-gather and reduce-scatter ungrouped")
    ap.add_argument("--no-extras", action="store_true", help="skip transport_local / ref_dtypes records")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    a = ap.parse_args(argv)
    a.warmup = max(a.warmup, 3)  # at least 3 untimed warm-up steps (the line reports the count run)
    return a


def dist_env():
    if "WORLD_SIZE" in os.environ and int(os.environ["WORLD_SIZE"]) > 1:
        return int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ.get("LOCAL_RANK", 0))
    return 0, 1, 0


def placement(args, world: int, ngpu_visible: int):
    """(n, devices of the ranks this process drives, n_gpus of the job, mode) or raises
    SystemExit(2) when the request cannot be honoured as asked."""
    if world > 1:  # torchrun: one rank per process, one GPU each
        if args.gpus != world:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; refusing to report n_gpus={world}")
        if args.ranks not in (0, world):
            raise SystemExit("bench.py: --ranks must equal WORLD_SIZE under torchrun (one rank per process)")
        return world, None, world, "torchrun"
    if args.gpus < 1:
        raise SystemExit("bench.py: --gpus must be >= 1")
    if args.gpus > ngpu_visible:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but only {ngpu_visible} GPU(s) visible")
    if args.gpus == 1:
        n = args.ranks or 8
        return n, [0] * n, 1, "local"
    n = args.ranks or args.gpus
    if n < args.gpus:
        raise SystemExit(f"bench.py: --ranks {n} < --gpus {args.gpus} would leave GPUs idle")
    return n, [r % args.gpus for r in range(n)], args.gpus, "one-process"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return PEAKS_FALLBACK, "fallback"


# ------------------------------------------------------------------ reference CPU path

def reference_time(n: int, chunk_bytes: int, seconds: float, mode: int = 1, max_steps: int = 10000,
                   warmup: int = 1):
    """The reference executor (oracle/_ref) on the host: run_allgather(int64) +
    run_reduce_scatter(float64, FloatSum) with equal bytes per chunk. The schedules and the
    reference's own Payload<T>s are built once (ref_prepare); a timed step calls only the
    reference's run_* (no marshalling, results dropped). Returns (seconds per step, steps, threads)."""
    import oracle as O

    R = O.ref()
    threads = os.cpu_count() or 1
    h = R.ref_prepare(n, O.max_trees(n), chunk_bytes // 8, mode, threads)
    if not h:
        raise RuntimeError(R.ref_last_error().decode())
    try:
        for _ in range(warmup):
            assert R.ref_run_prepared(h, 3) == 0
        steps, t0 = 0, time.perf_counter()
        while True:
            assert R.ref_run_prepared(h, 3) == 0
            steps += 1
            el = time.perf_counter() - t0
            if el >= seconds or steps >= max_steps:
                break
    finally:
        R.ref_free_prepared(h)
    return el / steps, steps, threads if mode else 1


def dbg(msg: str) -> None:
    if os.environ.get("BENCH_DEBUG"):
        print(f"[bench {os.environ.get('RANK', '0')}] {msg}", file=sys.stderr, flush=True)


def busbw_gbs(n: int, chunk_bytes: int, seconds: float) -> float:
    return 2.0 * n * (n - 1) * chunk_bytes / seconds / 1e9


# ------------------------------------------------------------------ clocks during the timed region

class ClockSampler:
    """NVML sampling of SM clock + throttle reasons every ~2 ms on the GPUs this process drives."""

    def __init__(self, devices):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.hs = [pynvml.nvmlDeviceGetHandleByIndex(d) for d in devices]
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.hs[0], pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            pass

    def _sample(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        for h in self.hs:
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                for k, bit in names.items():
                    if mask & bit:
                        self.reasons.add(k)
            except Exception:
                pass

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            time.sleep(0.002)

    def __enter__(self):
        if self.ok and not os.environ.get("BENCH_NO_CLOCKS"):
            self._sample()  # at least one sample inside a short timed region
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self.ok and hasattr(self, "_t"):
            self._stop.set()
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------ per-device graph plumbing

class Devices:
    """The GPUs this process drives: one dedicated stream each; CUDA graphs captured concurrently
    on every device (relaxed mode), replayed together, timed per device with events on the
    launching stream and reduced as the max over devices (then over ranks)."""

    def __init__(self, torch, devs, dist=None):
        self.torch, self.devs, self.dist = torch, list(devs), dist
        self.pre = None  # enqueued on the timing streams before the start events (time_ms)
        self.streams = {d: torch.cuda.Stream(d) for d in self.devs}

    def sync(self):
        for d in self.devs:
            self.torch.cuda.synchronize(d)

    def barrier(self):
        self.sync()
        if self.dist is not None:
            self.dist.barrier()
        self.sync()

    def capture(self, body):
        torch = self.torch
        graphs = {d: torch.cuda.CUDAGraph() for d in self.devs}
        for d in self.devs:
            self.streams[d].wait_stream(torch.cuda.current_stream(d))
            with torch.cuda.device(d):
                torch.cuda.set_stream(self.streams[d])
                graphs[d].capture_begin(capture_error_mode="relaxed")
        try:
            body()
        finally:
            for d in self.devs:
                with torch.cuda.device(d):
                    graphs[d].capture_end()
                    torch.cuda.set_stream(torch.cuda.default_stream(d))
        return graphs

    def replay(self, graphs):
        torch = self.torch
        for d in self.devs:
            with torch.cuda.device(d), torch.cuda.stream(self.streams[d]):
                graphs[d].replay()

    def events(self):
        E = self.torch.cuda.Event
        return {d: (E(enable_timing=True), E(enable_timing=True)) for d in self.devs}

    def time_ms(self, run):
        """barrier; device barrier; start events; run(); end events; barrier -> max over devices (ms).
        The device barrier (patCommBarrier on the timing streams, outside the timed region) lines
        the GPUs up, so host jitter in leaving the host barrier is not timed as collective time."""
        ev = self.events()
        self.barrier()
        if self.pre is not None:
            self.pre()
        for d in self.devs:
            ev[d][0].record(self.streams[d])
        run()
        for d in self.devs:
            ev[d][1].record(self.streams[d])
        self.barrier()
        return max(ev[d][0].elapsed_time(ev[d][1]) for d in self.devs)


def max_over_ranks(torch, dist, dev, values):
    t = torch.tensor(values, dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.tolist()]


# ------------------------------------------------------------------ PAT arm

def run_pat(args, rank, world, local):
    import torch

    dist = None
    n, devices, n_gpus, mode = placement(args, world, torch.cuda.device_count())
    from paper_2506_20252_b200 import FLOAT32, FLOAT64, INT64, SUM, PatComm
    from paper_2506_20252_b200._lib import lib

    C = args.chunk_bytes
    elems = C // 4
    if mode == "torchrun":
        import torch.distributed as dist

        share = os.environ.get("BENCH_SHARE_GPUS") == "1"
        if share:  # rehearsal of the N-process path on fewer GPUs (NCCL refuses two ranks per GPU)
            local %= torch.cuda.device_count()
            args.no_nccl = True
        dev0 = torch.device(f"cuda:{local}")
        torch.cuda.set_device(dev0)
        os.environ.setdefault("NCCL_ALGO", "Ring")  # affects only the NCCL comparison below
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev0)
        devices = [local]
        comm = PatComm.from_process_group(device=local)
        desc = f"{n} ranks on {n} GPUs (torchrun: 1 process per GPU, CUDA IPC inbox pools)"
    else:
        torch.cuda.set_device(devices[0])
        comm = PatComm.init_all(n, devices)
        desc = (f"{n} logical ranks on 1 GPU (fused single-device executor, local.cu)" if mode == "local" else
                f"{n} ranks on {n_gpus} GPUs, one process (patCommInitAll), devices {devices}")
    dev0 = torch.device(f"cuda:{devices[0]}")
    L = len(devices)  # ranks this process drives
    D = Devices(torch, sorted(set(devices)), dist)
    streams = [D.streams[d] for d in devices]

    # 2x L2 of scratch per GPU, read before every timed region (leaves L2 clean: the dirty output
    # lines of the previous region are written back before the clock starts, not inside it)
    flush = {d: torch.empty(2 * L2_BYTES // 4, device=f"cuda:{d}") for d in D.devs}

    def pre():
        # L2 flush by reads, device barrier (GPUs aligned), then a ~100 us spin on each timing
        # stream so the graph replays are queued behind it before the start events: neither host
        # jitter between ranks nor the host's graph-launch latency is timed as collective time
        for d in D.devs:
            with torch.cuda.device(d), torch.cuda.stream(D.streams[d]):
                flush[d].sum()
        comm.barrier(streams)
        for d in D.devs:
            with torch.cuda.device(d), torch.cuda.stream(D.streams[d]):
                torch.cuda._sleep(int(os.environ.get("BENCH_SLEEP_CYCLES", "200000")))
    D.pre = pre
    pre()  # loads the flush / spin kernels' modules now (lazy loading), not inside a timed region's prologue
    D.barrier()
    g = {d: torch.Generator(device=f"cuda:{d}").manual_seed(1234 + 17 * rank + d) for d in D.devs}

    def rnd(numel, d):
        return torch.rand(numel, device=f"cuda:{d}", generator=g[d])

    # Inputs larger than L2: the step's buffers are rotated over S sets whose total per GPU
    # exceeds twice the 126 MB L2, so every timed step starts cold.
    per_gpu_ranks = max(devices.count(d) for d in D.devs)
    step_bytes = per_gpu_ranks * 2 * (n + 1) * C
    S = max(2, -(-(2 * L2_BYTES) // step_bytes) + 1)
    sets = []
    for _ in range(S):
        sets.append({
            "ag_send": [rnd(elems, d) for d in devices],
            "ag_recv": [torch.empty(n * elems, device=f"cuda:{d}") for d in devices],
            "rs_send": [rnd(n * elems, d) for d in devices],
            "rs_recv": [torch.empty(elems, device=f"cuda:{d}") for d in devices],
        })

    def call(c, kinds, bs, dtype=FLOAT32, count=elems):
        # a step ("ag", "rs") is one group (patGroupStart/End): the all-gather and the reduce-scatter
        # run as one launch; "ungrouped" issues them one after the other
        grouped = "ag" in kinds and "rs" in kinds and "ungrouped" not in kinds and not args.no_group
        if grouped:
            lib().patGroupStart()
        try:
            if "ag" in kinds:
                c.all_gather(bs["ag_send"], bs["ag_recv"], count, dtype, streams=streams)
            if "rs" in kinds:
                c.reduce_scatter(bs["rs_send"], bs["rs_recv"], count, dtype, SUM, streams=streams)
        finally:
            if grouped:
                rc = lib().patGroupEnd()
                if rc:
                    raise RuntimeError(f"patGroupEnd: {rc}")

    dbg("warmup")
    for _ in range(args.warmup):
        for bs in sets:
            call(comm, ("ag", "rs"), bs)
    D.barrier()
    comm.raise_async_error()

    # The timed region replays CUDA graphs holding exactly K steps (step k = PAT all-gather +
    # PAT reduce-scatter on buffer set k % S), captured from the C-ABI calls: the launches are
    # the library's own kernels back to back, without Python/ctypes host gaps. More graphs of K
    # all-gathers and K reduce-scatters give the per-collective latencies.
    K = args.steps
    G = min(K, 1000)  # steps per graph; the timed region replays it K // G times (+ a remainder graph)
    rem = K % G

    def graphs_for(c, kinds, sets_=sets, **kw):
        def body(count):
            def run():
                for k in range(count):
                    call(c, kinds, sets_[k % len(sets_)], **kw)
            return run
        full = D.capture(body(G))
        part = D.capture(body(rem)) if rem else None
        return full, part

    def replay_k(pair):
        full, part = pair

        def run():
            for _ in range(K // G):
                D.replay(full)
            if part is not None:
                D.replay(part)
        return run

    dbg("capture")
    graphs = {kinds: graphs_for(comm, kinds) for kinds in (("ag", "rs"), ("ag", "rs", "ungrouped"), ("ag",), ("rs",))}
    for pair in graphs.values():  # warm replay
        replay_k(pair)()
    D.barrier()

    dbg("timed")
    with ClockSampler(D.devs) as clocks:
        step_ms = D.time_ms(replay_k(graphs[("ag", "rs")]))
        if os.environ.get("BENCH_TRIALS"):  # diagnostics: more timed regions of the same K steps
            extra = [D.time_ms(replay_k(graphs[("ag", "rs")])) for _ in range(int(os.environ["BENCH_TRIALS"]))]
            dbg(f"step trials (us/step): {[round(1e3 * x / K, 2) for x in [step_ms] + extra]}")
        ag_ms = D.time_ms(replay_k(graphs[("ag",)]))
        rs_ms = D.time_ms(replay_k(graphs[("rs",)]))
        step_ung_ms = D.time_ms(replay_k(graphs[("ag", "rs", "ungrouped")]))
    comm.raise_async_error()
    step_ms, ag_ms, rs_ms, step_ung_ms = max_over_ranks(torch, dist, dev0, [step_ms, ag_ms, rs_ms, step_ung_ms])
    del graphs
    ms_per_step = step_ms / K
    value = busbw_gbs(n, C, ms_per_step / 1e3)

    # ---- the same calls launched eagerly (no graphs) through the Python binding: K back-to-back
    # calls per collective, events around the K (as the NCCL comparison is timed)
    def eager_k(kinds):
        def run():
            for k in range(K):
                call(comm, kinds, sets[k % S])
        return run
    eager_bb = max_over_ranks(torch, dist, dev0, [D.time_ms(eager_k(("ag",))), D.time_ms(eager_k(("rs",))),
                                                   D.time_ms(eager_k(("ag", "rs")))])
    # ---- isolated eager calls (events per call on an idle stream: host submission included)
    KE = min(K, 100)
    eev = [D.events() for _ in range(3 * KE)]
    D.barrier()
    for k in range(KE):
        bs = sets[k % S]
        for d in D.devs:
            eev[3 * k][d][0].record(D.streams[d])
        call(comm, ("ag",), bs)
        for d in D.devs:
            eev[3 * k][d][1].record(D.streams[d])
            eev[3 * k + 1][d][0].record(D.streams[d])
        call(comm, ("rs",), bs)
        for d in D.devs:
            eev[3 * k + 1][d][1].record(D.streams[d])
    D.barrier()
    ag_e = max(sum(eev[3 * k][d][0].elapsed_time(eev[3 * k][d][1]) for k in range(KE)) for d in D.devs)
    rs_e = max(sum(eev[3 * k + 1][d][0].elapsed_time(eev[3 * k + 1][d][1]) for k in range(KE)) for d in D.devs)
    ag_e, rs_e = max_over_ranks(torch, dist, dev0, [ag_e, rs_e])
    eager_iso_us = {"all_gather": 1e3 * ag_e / KE, "reduce_scatter": 1e3 * rs_e / KE,
                    "timing": "one eager call at a time on an idle GPU, events around each call: includes the "
                              "host's submission time (Python binding + C ABI)"}
    eager_us = {"all_gather": 1e3 * eager_bb[0] / K, "reduce_scatter": 1e3 * eager_bb[1] / K,
                "step": 1e3 * eager_bb[2] / K,
                "timing": "K back-to-back eager calls (steps: grouped) through the Python binding, events around the K"}

    dbg("e2e")
    # ---- e2e through the C ABI with host buffers (pinned), H2D + D2H inside the timed region.
    # Rotating device sets (3 or 4 per device): step k's inputs go up on a copy stream into set k % NB
    # while step k-1 runs, and step k-1's results come down on another copy stream (PCIe is full
    # duplex); every step still copies all of its inputs in and its results out inside the
    # timed region.
    # buffers: per device ONE pinned host block and ONE device block per direction, [all-gather |
    # reduce-scatter] x the device's ranks, so every step moves each device's inputs in one H2D copy
    # and its results in one D2H copy (fewer, larger PCIe transfers)
    E = max(3, min(K, 20))
    # step k+1's upload, step k's compute and step k-1's download all in flight (double buffering
    # left PCIe idle ~17% of a step: tools/e2e_probe.py, 2.04 vs 1.71 ms; a 4th set: 39.9 -> 44.5
    # GB/s at N=2, 90 -> 123 at N=4, profiles/r02_e2e_sets.txt)
    ranks_on = {d: [i for i, di in enumerate(devices) if di == d] for d in D.devs}
    # 4 sets for small steps, 3 when a device moves >= 32 MiB a step (N=1: 68 vs 64 GB/s on one box;
    # N=2 one process: 30 vs 26; profiles/r02_e2e_sets.txt)
    big = max(len(v) for v in ranks_on.values()) * (n + 1) * C >= 32 << 20
    NB = int(os.environ.get("BENCH_E2E_BUFFERS", "3" if big else "4"))

    def blocks(mk):
        """{"in": {d: block}, "out": {d: block}, ag_send/rs_send/ag_recv/rs_recv: per-rank views}"""
        b = {"in": {}, "out": {}, "ag_send": [None] * L, "rs_send": [None] * L, "ag_recv": [None] * L,
             "rs_recv": [None] * L}
        for d, idx in ranks_on.items():
            m = len(idx)
            bi, bo = mk(d, m * (1 + n) * elems), mk(d, m * (n + 1) * elems)
            b["in"][d], b["out"][d] = bi, bo
            for j, i in enumerate(idx):
                b["ag_send"][i] = bi[j * elems:(j + 1) * elems]
                b["rs_send"][i] = bi[m * elems + j * n * elems:m * elems + (j + 1) * n * elems]
                b["ag_recv"][i] = bo[j * n * elems:(j + 1) * n * elems]
                b["rs_recv"][i] = bo[m * n * elems + j * elems:m * n * elems + (j + 1) * elems]
        return b

    hb = blocks(lambda d, sz: torch.empty(sz, dtype=torch.float32).pin_memory())
    for i in range(L):
        hb["ag_send"][i].copy_(sets[0]["ag_send"][i].cpu())
        hb["rs_send"][i].copy_(sets[0]["rs_send"][i].cpu())
    dsets = [blocks(lambda d, sz: torch.empty(sz, device=f"cuda:{d}")) for _ in range(NB)]
    for bs in dsets:  # untimed first use of the new buffers
        call(comm, ("ag", "rs"), bs)
    s_in = {d: torch.cuda.Stream(d) for d in D.devs}
    s_out = {d: torch.cuda.Stream(d) for d in D.devs}
    ev = lambda: {d: torch.cuda.Event() for d in D.devs}  # noqa: E731
    h2d_done, comp_done, d2h_done = [ev() for _ in range(E)], [ev() for _ in range(E)], [ev() for _ in range(E)]
    e01 = D.events()
    D.barrier()
    for d in D.devs:
        e01[d][0].record(D.streams[d])
        s_in[d].wait_stream(D.streams[d])
        s_out[d].wait_stream(D.streams[d])
    t_host = time.perf_counter()
    for k in range(E):
        bs = dsets[k % NB]
        for d in D.devs:
            with torch.cuda.device(d), torch.cuda.stream(s_in[d]):
                if k >= NB:
                    s_in[d].wait_event(comp_done[k - NB][d])  # set k % NB's inputs are free
                bs["in"][d].copy_(hb["in"][d], non_blocking=True)
                h2d_done[k][d].record(s_in[d])
            D.streams[d].wait_event(h2d_done[k][d])
            if k >= NB:
                D.streams[d].wait_event(d2h_done[k - NB][d])  # set k % NB's outputs were read back
        call(comm, ("ag", "rs"), bs)
        for d in D.devs:
            comp_done[k][d].record(D.streams[d])
            with torch.cuda.device(d), torch.cuda.stream(s_out[d]):
                s_out[d].wait_event(comp_done[k][d])
                hb["out"][d].copy_(bs["out"][d], non_blocking=True)
                d2h_done[k][d].record(s_out[d])
    for d in D.devs:
        D.streams[d].wait_event(d2h_done[E - 1][d])
        D.streams[d].wait_event(h2d_done[E - 1][d])
        e01[d][1].record(D.streams[d])
    e2e_host_us = 1e6 * (time.perf_counter() - t_host) / E  # host submission time per step
    D.barrier()
    e2e_ms = max_over_ranks(torch, dist, dev0, [max(e01[d][0].elapsed_time(e01[d][1]) for d in D.devs) / E])[0]
    # the host copies of the last step's results equal the device results of the same inputs
    # (sets[0], timed above): a wrong or partial copy-out fails the run instead of being timed
    for i in range(L):
        if not (torch.equal(hb["ag_recv"][i], sets[0]["ag_recv"][i].cpu()) and
                torch.equal(hb["rs_recv"][i], sets[0]["rs_recv"][i].cpu())):
            raise RuntimeError(f"e2e: rank slot {i}: host results differ from the device results")
    # bytes of the whole job per step (every rank's inputs up, every rank's outputs down)
    ranks_total = n
    h2d = ranks_total * (elems + n * elems) * 4
    d2h = ranks_total * (n * elems + elems) * 4

    # ---- NCCL Ring comparison (torchrun), timed exactly like the PAT arm: CUDA graphs of K steps
    nccl = None
    dbg("nccl")
    if mode == "torchrun" and not args.no_nccl:
        def nccl_call(kinds, bs):
            if "ag" in kinds:
                dist.all_gather_into_tensor(bs["ag_recv"][0], bs["ag_send"][0])
            if "rs" in kinds:
                dist.reduce_scatter_tensor(bs["rs_recv"][0], bs["rs_send"][0])

        for _ in range(args.warmup):
            for bs in sets:
                with torch.cuda.stream(streams[0]):
                    nccl_call(("ag", "rs"), bs)
        D.barrier()
        timing = "graph"
        try:
            if not args.nccl_graph:  # capturing NCCL inside this process hangs (r02, 2 GPUs, both with
                raise RuntimeError("eager")  # raw capture and torch.cuda.graph): eager; graph-mode NCCL is in bench_sweep.py
            def nbody(kinds, count):
                def run():
                    for k in range(count):
                        nccl_call(kinds, sets[k % S])
                return run
            def ncapture(body):  # as bench_sweep.py: torch.cuda.graph (global capture mode) on the timing stream
                d = devices[0]
                g_ = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g_, stream=D.streams[d]):
                    body()
                return {d: g_}
            ngraphs = {}
            for kinds in (("ag", "rs"), ("ag",), ("rs",)):
                ngraphs[kinds] = (ncapture(nbody(kinds, G)), ncapture(nbody(kinds, rem)) if rem else None)
            for pair in ngraphs.values():
                replay_k(pair)()
            D.barrier()
            nt = [D.time_ms(replay_k(ngraphs[kinds])) for kinds in (("ag", "rs"), ("ag",), ("rs",))]
            del ngraphs
        except Exception as e:  # eager fallback, labelled
            dbg(f"nccl graph capture skipped/failed: {e}")
            timing = ("eager: K back-to-back calls on one stream (GPU-bound: NCCL's host launch is shorter than "
                      "its kernel); CUDA graphs of NCCL calls hang inside bench.py, see --nccl-graph"
                      if str(e) == "eager" else f"eager (graph capture failed: {type(e).__name__})")
            D.barrier()

            def eager(kinds):
                def run():
                    with torch.cuda.stream(streams[0]):
                        for k in range(K):
                            nccl_call(kinds, sets[k % S])
                return run
            nt = [D.time_ms(eager(kinds)) for kinds in (("ag", "rs"), ("ag",), ("rs",))]
        nt = max_over_ranks(torch, dist, dev0, nt)
        nccl = {"algo": os.environ.get("NCCL_ALGO"), "ms_per_step": nt[0] / K,
                "busbw_gbs": busbw_gbs(n, C, nt[0] / K / 1e3),
                "ag_us": 1e3 * nt[1] / K, "rs_us": 1e3 * nt[2] / K,
                "nccl_version": ".".join(str(x) for x in torch.cuda.nccl.version()), "timing": timing,
                "pat_speedup_step": nt[0] / step_ms,
                "pat_speedup_step_ungrouped": nt[0] / step_ung_ms,
                "pat_eager_ms_per_step": eager_bb[2] / K,
                "pat_speedup_step_eager": nt[0] / eager_bb[2],
                "note": "NCCL is timed eagerly (K back-to-back calls); pat_speedup_step_eager compares PAT timed "
                        "the same way (eager grouped steps). NCCL's all-gather and reduce-scatter run one after "
                        "the other (torch.distributed cannot coalesce two different collectives); "
                        "pat_speedup_step_ungrouped compares the same call sequence from CUDA graphs, "
                        "pat_speedup_step PAT's grouped launch"}

    # ---- N = 1 extras: the same n = 8 workload through the PAT transport kernel (per-round
    # messages through the inbox pools with flags), and the repo at the reference arm's dtypes
    extras = {}
    if mode == "local" and not args.no_extras:
        dbg("transport_local")
        tcomm = PatComm.init_all(n, devices, fused=-1)
        for _ in range(max(3, args.warmup // 4)):
            for bs in sets:
                call(tcomm, ("ag", "rs"), bs)
        D.barrier()
        tg = {kinds: graphs_for(tcomm, kinds) for kinds in (("ag",), ("rs",))}
        for pair in tg.values():
            replay_k(pair)()
        t_ag = D.time_ms(replay_k(tg[("ag",)]))
        t_rs = D.time_ms(replay_k(tg[("rs",)]))
        tcomm.raise_async_error()
        pa, pr = tcomm.plan(0, elems, FLOAT32), tcomm.plan(1, elems, FLOAT32)
        names = {1: "LL", 2: "SIMPLE", 3: "PULL", 5: "LL32"}
        extras["transport_local"] = {
            "kernel": "pat_kernel (fused = -1)", "all_gather_us": 1e3 * t_ag / K, "reduce_scatter_us": 1e3 * t_rs / K,
            "protocol": {"all_gather": names.get(pa["protocol"]), "reduce_scatter": names.get(pr["protocol"])},
            "channels": pa["channels"], "rounds": pa["rounds"], "pool_bytes_per_rank": pa["pool_bytes"],
            "busbw_gbs": busbw_gbs(n, C, (t_ag + t_rs) / K / 1e3),
            "timing": "CUDA graphs of K calls per collective, same buffer sets"}
        del tg
        tcomm.destroy()
        # int64 all-gather + float64 reduce-scatter at equal bytes: the reference arm's dtypes
        dbg("ref_dtypes")
        e8 = C // 8
        for _ in range(2):
            for bs in sets:
                call(comm, ("ag",), bs, dtype=INT64, count=e8)
                call(comm, ("rs",), bs, dtype=FLOAT64, count=e8)
        D.barrier()
        rg_f = graphs_for(comm, ("rs",), dtype=FLOAT64, count=e8)
        rg_a = graphs_for(comm, ("ag",), dtype=INT64, count=e8)
        for pair in (rg_f, rg_a):
            replay_k(pair)()
        t_a = D.time_ms(replay_k(rg_a))
        t_f = D.time_ms(replay_k(rg_f))
        extras["ref_dtypes"] = {
            "dtype": "int64 all-gather + f64 reduce-scatter(sum), equal bytes (the reference arm's dtypes)",
            "ms_per_step": (t_a + t_f) / K, "value": busbw_gbs(n, C, (t_a + t_f) / K / 1e3), "unit": "GB/s",
            "all_gather_us": 1e3 * t_a / K, "reduce_scatter_us": 1e3 * t_f / K,
            "timing": "sum of CUDA-graph-timed K int64 all-gathers and K f64 reduce-scatters"}
        del rg_f, rg_a

    # ---- roofline of the dominant kernel
    peaks, peak_src = load_peaks()
    dom = "reduce_scatter" if rs_ms >= ag_ms else "all_gather"
    dom_us = 1e3 * max(ag_ms, rs_ms) / K
    if mode == "local":
        # local mode: read n*C + write n^2*C (AG) / read n^2*C + write n*C (RS) per collective; a
        # grouped step is ONE launch (local_group_kernel) doing both, and it is the step's kernel
        coll_bytes = (n * n + n) * C
        peak = float(peaks.get("hbm_gbs", PEAKS_FALLBACK["hbm_gbs"]))
        per_coll = {c_: {"kernel": k_, "us": 1e3 * t_ / K, "frac": coll_bytes / (t_ / K * 1e-3) / 1e9 / peak}
                    for c_, k_, t_ in (("all_gather", "local_ag32_kernel", ag_ms),
                                       ("reduce_scatter", "local_rs_flat_kernel", rs_ms))}
        if not args.no_group:
            algo_bytes, dom_us = 2 * coll_bytes, 1e3 * step_ms / K
            kern = "local_group_kernel (the grouped step: all-gather + reduce-scatter in one launch)"
        else:
            algo_bytes = coll_bytes
            kern = "local_rs_flat_kernel" if dom == "reduce_scatter" else "local_ag32_kernel"
        roof = {"bound": "hbm", "kernel": kern, "unit": "GB/s", "algorithmic_bytes_per_launch": algo_bytes,
                "peak_source": f"{peak_src} MEASURED_PEAKS.json hbm_gbs", "per_collective": per_coll}
        achieved = algo_bytes / (dom_us * 1e-6) / 1e9
        # live ceilings for the same byte counts, K launches over 4 rotating buffers (> 2x L2):
        # a copy (the grouped step's 50/50 read/write mix) and a fill (the all-gather is write-bound)
        nel = coll_bytes // 4
        cbufs = [torch.empty(nel, device=dev0) for _ in range(8)]
        for b_ in cbufs:
            b_.fill_(0.0)
        D.sync()

        def copies():
            with torch.cuda.stream(D.streams[devices[0]]):
                for k in range(K):
                    cbufs[2 * (k % 4) + 1].copy_(cbufs[2 * (k % 4)])

        def fills():
            with torch.cuda.stream(D.streams[devices[0]]):
                for k in range(K):
                    cbufs[k % 4].fill_(float(k))
        copies()  # warm: lazy module loading of the copy kernel
        fills()
        D.sync()
        copy_ms = D.time_ms(copies)
        fill_ms = D.time_ms(fills)
        cgbs = 2 * coll_bytes / (copy_ms / K * 1e-3) / 1e9
        wgbs = coll_bytes / (fill_ms / K * 1e-3) / 1e9
        roof["copy_ceiling"] = {"gbs": cgbs, "frac_of_peak": cgbs / peak, "us": 1e3 * copy_ms / K,
                                "kernel": "torch copy_ of 72 MiB (144 MiB of traffic), K launches"}
        roof["write_ceiling"] = {"gbs": wgbs, "frac_of_peak": wgbs / peak, "us": 1e3 * fill_ms / K,
                                 "kernel": "torch fill_ of 72 MiB (write-only), K launches"}
        del cbufs
    else:
        # per GPU: every rank on it receives (n-1)*C over NVLink per launch (ranks sharing a GPU
        # share its links, so the GPU's ingress is ranks_on_gpu * (n-1) * C minus what stays local)
        coll_bytes = (n - 1) * C
        peak = NVLINK_PEER_COPY_GBS
        per_coll = {c_: {"kernel": "pat_kernel", "us": 1e3 * t_ / K,
                         "frac": coll_bytes / (t_ / K * 1e-3) / 1e9 / peak}
                    for c_, t_ in (("all_gather", ag_ms), ("reduce_scatter", rs_ms))}
        if not args.no_group:  # the timed step is one grouped launch carrying both collectives
            algo_bytes, dom_us = 2 * coll_bytes, 1e3 * step_ms / K
            kern = "pat_group_kernel (the grouped step: all-gather + reduce-scatter in one launch)"
        else:
            algo_bytes, kern = coll_bytes, f"pat_kernel ({dom})"
        roof = {"bound": "nvlink", "kernel": kern, "unit": "GB/s",
                "algorithmic_bytes_per_launch": algo_bytes, "per_collective": per_coll,
                "peak_source": "measured NVLink peer copy 770 GB/s per direction (B200_PROFILING.md)"}
        achieved = algo_bytes / (dom_us * 1e-6) / 1e9
        roof["frac_of_nominal_900"] = achieved / NVLINK_NOMINAL_GBS
        roof["frac_of_sm_push_704"] = achieved / NVLINK_SM_PUSH_GBS
    roof.update({"achieved": achieved, "peak": peak, "frac": achieved / peak, "traffic": None,
                 "launch_us": dom_us})
    if "copy_ceiling" in roof and not args.no_group:
        roof["frac_of_copy_ceiling"] = achieved / roof["copy_ceiling"]["gbs"]
    if "write_ceiling" in roof:
        roof["per_collective"]["all_gather"]["frac_of_write_ceiling"] = (
            coll_bytes / (ag_ms / K * 1e-3) / 1e9 / roof["write_ceiling"]["gbs"])
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            tr = json.load(open(tpath))
            key = (f"{'local' if mode == 'local' else 'nvlink'}_n{n}_group" if not args.no_group else
                   f"{'local' if mode == 'local' else 'nvlink'}_n{n}_{dom}")
            if key in tr:
                roof["traffic"] = tr[key]["dram_bytes_per_launch"]
                roof["traffic_source"] = tr[key].get("source")
                if "nvlink_tx_bytes_per_launch" in tr[key]:  # NVLink egress of the same ncu launch
                    roof["nvlink_tx_bytes"] = tr[key]["nvlink_tx_bytes_per_launch"]
                    if "nvlink_tx_user_bytes_per_launch" in tr[key]:
                        roof["nvlink_tx_user_bytes"] = tr[key]["nvlink_tx_user_bytes_per_launch"]
        except Exception:
            pass

    # small messages are latency-bound: compare with the PAT step floor — the zero-byte time of
    # R = ceil(log2 n) polling rounds (LL, the lowest fixed cost of the cost-model fit,
    # profiles/r01f_costmodel_fit.json) plus the payload on the wire with LL32's one flag word
    # per 28 bytes, at the measured two-way SM-push ceiling (profiles/r01_bidir_probe_g4.txt)
    lat_floor = None
    if mode != "local":
        plan = comm.plan(0, elems, FLOAT32)
        R = plan["rounds"]
        zero_us = 3.41 + 1.40 * R
        wire_us = (32.0 / 28.0) * (n - 1) * C / (NVLINK_SM_PUSH_GBS * 1e3)
        lat_floor = {"rounds": R, "protocol": plan["protocol"], "zero_byte_us": zero_us,
                     "wire_us_at_704gbs": wire_us, "floor_us": zero_us + wire_us, "achieved_us": 1e3 * ag_ms / K,
                     "frac": (zero_us + wire_us) / (1e3 * ag_ms / K),
                     "source": "profiles/r01f_costmodel_fit.json (LL a, b), profiles/r01_bidir_probe_g4.txt"}
        if not args.no_group:  # the grouped step: one fixed cost, both collectives' bytes on the wire
            lat_floor["grouped_step"] = {"floor_us": zero_us + 2 * wire_us, "achieved_us": 1e3 * step_ms / K,
                                         "frac": (zero_us + 2 * wire_us) / (1e3 * step_ms / K)}

    clk = clocks.summary()
    if dist is not None:
        allc = [None] * world
        dist.all_gather_object(allc, clk)
        clk = {"sm_mhz": statistics.median([c["sm_mhz"] for c in allc if c["sm_mhz"]] or [0]),
               "sm_max_mhz": allc[0]["sm_max_mhz"], "reasons": sorted({r for c in allc for r in c["reasons"]}),
               "samples": sum(c["samples"] for c in allc)}

    plan_ag = comm.plan(0, elems, FLOAT32)
    plan_rs = comm.plan(1, elems, FLOAT32)
    pool_info = comm.pool_info()
    out = None
    if rank == 0:
        cpu = None
        if n_gpus == 1 and not args.no_cpu_baseline:
            try:
                sec, steps, thr = reference_time(n, C, args.cpu_seconds)
                cpu = {"value": busbw_gbs(n, C, sec), "unit": "GB/s", "cores": thr, "kind": "reference",
                       "ms_per_step": sec * 1e3,
                       "sample": f"{steps} steps of the reference executor (oracle/_ref = /root/reference/proj/src "
                                 f"compiled), n={n}, {C} B/rank, run_allgather(int64)+run_reduce_scatter(f64) on "
                                 f"payloads built once, ExecMode::Parallel x{thr} threads, {args.cpu_seconds:.0f} s budget"}
            except Exception as e:  # the reference library must be built in-tree
                cpu = {"value": None, "unit": "GB/s", "cores": 0, "kind": "reference", "sample": f"unavailable: {e}"}
        launches_per_gpu = (1 if not args.no_group else 2) * K  # a grouped step is one launch per GPU
        out = {
            "metric": "PAT all-gather + reduce-scatter(sum) aggregate bus bandwidth, 1 MiB fp32 per rank",
            "value": value, "unit": "GB/s", "n_gpus": n_gpus, "steps": K, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (torch.rand on device)",
            "config": {"workload": ("BASELINE configs[0]: PAT AG + RS(sum), n=8, 1 MiB fp32 per rank" if n == 8 else
                                    f"BASELINE configs[0] shape at n={n}: PAT AG + RS(sum), 1 MiB fp32 per rank"),
                       "nranks": n, "mode": mode, "placement": desc, "chunk_bytes": C, "trees": plan_ag["trees"],
                       "rounds": plan_ag["rounds"],
                       "l2": f"inputs larger than L2: {S} rotating buffer sets, {S * step_bytes / 2**20:.0f} MiB per GPU",
                       "timing": "CUDA events around CUDA-graph replays of exactly K steps (captured C-ABI calls), "
                                 "max over devices and ranks",
                       "plan_allgather": plan_ag, "plan_reduce_scatter": plan_rs},
            "latency_us": {"all_gather": 1e3 * ag_ms / K, "reduce_scatter": 1e3 * rs_ms / K,
                           "timing": "graph of K back-to-back calls per collective"},
            "step_grouped": not args.no_group,
            "ms_per_step_ungrouped": step_ung_ms / K,
            "value_ungrouped": busbw_gbs(n, C, step_ung_ms / K / 1e3),
            "latency_us_eager": eager_us,
            "latency_us_eager_isolated": eager_iso_us,
            "e2e": {"value": busbw_gbs(n, C, e2e_ms / 1e3), "unit": "GB/s", "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "host_submit_us_per_step": e2e_host_us,
                    "path": "pinned host -> device copies, patAllGather + patReduceScatter (C ABI), device -> host; "
                            f"{NB} rotating device sets: step k+1 uploads while step k-1 downloads (PCIe full duplex); one H2D and one D2H copy "
                            "per device per step"},
            "gpu_launches": launches_per_gpu * n_gpus,
            "gpu_launches_per_gpu": launches_per_gpu,
            "roofline": roof,
            "latency_floor": lat_floor,
            "cpu_baseline": cpu,
            "clocks": clk,
            "staging": pool_info,
        }
        if nccl:
            out["nccl_ring"] = nccl
        if mode == "torchrun" and os.environ.get("BENCH_SHARE_GPUS") == "1":
            out["rehearsal"] = f"BENCH_SHARE_GPUS: {n} processes on {torch.cuda.device_count()} GPUs, not a bench value"
        out.update(extras)
    comm.destroy()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return out


def run_reference(args, rank, world):
    if rank != 0:
        return None
    n = world if world > 1 else (args.ranks or (8 if args.gpus == 1 else args.gpus))
    C = args.chunk_bytes
    # W warm-up steps (at most 3: each is the whole workload, ~90 ms), then exactly K timed steps
    # unless K steps would exceed ~2 minutes of host time: then as many as fit, reported in
    # "steps" and in the sample description
    est, _, _ = reference_time(n, C, 0.0, max_steps=1, warmup=min(args.warmup, 3))
    timed = max(1, min(args.steps, int(120.0 / max(est, 1e-6))))
    sec, steps, thr = reference_time(n, C, 1e9, max_steps=timed, warmup=0)
    budget = sec * steps
    value = busbw_gbs(n, C, sec)
    return {"impl": "reference", "metric": "PAT all-gather + reduce-scatter(sum) aggregate bus bandwidth, 1 MiB fp32 per rank",
            "value": value, "unit": "GB/s", "n_gpus": world if world > 1 else args.gpus, "steps": steps,
            "warmup": args.warmup,
            "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "int64 AG + f64 RS (equal bytes)", "data": "synthetic (reference mt19937_64 payloads)",
            "config": {"workload": ("BASELINE configs[0]: PAT AG + RS(sum), n=8, 1 MiB per rank" if n == 8 else
                                    f"BASELINE configs[0] shape at n={n}: PAT AG + RS(sum), 1 MiB per rank"),
                       "nranks": n, "chunk_bytes": C, "placement": "in-process ranks on host cores"},
            "cpu_baseline": {"value": value, "unit": "GB/s", "cores": thr, "kind": "reference",
                             "sample": f"{steps} timed steps (of --steps {args.steps}) of the whole workload, "
                                       f"payloads built once (ref_prepare), ExecMode::Parallel x{thr} threads, {budget:.1f} s"},
            "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    args = parse()
    # one JSON line on stdout: everything else (NCCL banners, warnings) goes to stderr
    real_stdout = os.dup(1)
    os.dup2(2, 1)
    sys.stdout = os.fdopen(os.dup(2), "w")
    rank, world, local = dist_env()
    try:
        if args.impl == "reference":
            out = run_reference(args, rank, world)
        else:
            out = run_pat(args, rank, world, local)
    except SystemExit as e:
        if isinstance(e.code, str):
            print(e.code, file=sys.stderr, flush=True)
            os._exit(2)
        raise
    if rank == 0 and out is not None:
        if args.impl == "pat" and out["n_gpus"] != args.gpus:  # never report a different GPU count
            print(f"bench.py: measured n_gpus={out['n_gpus']} != --gpus {args.gpus}", file=sys.stderr)
            os._exit(2)
        with os.fdopen(real_stdout, "w") as f:
            f.write(json.dumps(out) + "\n")


if __name__ == "__main__":
    main()
