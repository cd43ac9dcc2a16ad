"""Extract the judged metrics of an ncu report into a small CSV (run where ncu is installed).

  python tools/summarize_ncu.py gpurun_out/prof_local_fused.ncu-rep profiles/r01_ncu_local_fused.csv
"""
import csv
import io
import subprocess
import sys

METRICS = [
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "smsp__warp_issue_stalled_membar_per_warp_active.pct", "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
]


def main(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    idx = [head.index(m) for m in METRICS if m in head]
    with open(out, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow([head[i] + (f" [{units[i]}]" if units[i] else "") for i in idx])
        for r in rows[2:]:
            w.writerow([r[i] for i in idx])
    print(open(out).read())


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
