"""Summarize an ncu NVLink capture of tools/ncu_nvlink.py (one row per profiled launch).

  python tools/summarize_nvlink.py gpurun_out/ncu_nvlink_g4.csv --log gpurun_out/ncu_nv4.log > profiles/r01f_ncu_nvlink_g4.txt

Per launch: duration, NVLink bytes sent / received (all, and user payload), the achieved egress
GB/s (payload and on the wire) and the wire overhead (packet headers, request/response protocol).
Egress is the clean figure: the profiled device's own stores all fall inside its kernel, while
its peers (launched first, unprofiled) may have pushed some of its ingress before it started.
"""
import argparse
import csv
import re
from collections import defaultdict


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--log", default=None, help="tools/ncu_nvlink.py stdout (case names)")
    args = ap.parse_args()
    rows = [r for r in csv.reader(l for l in open(args.csv) if not l.startswith("=="))]
    h = rows[0]
    ii, ki, mi, vi = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    d = defaultdict(dict)
    for r in rows[1:]:
        d[int(r[ii])][r[mi]] = float(r[vi].replace(",", ""))
        d[int(r[ii])]["kernel"] = r[ki]
    cases = []
    if args.log:
        for line in open(args.log):
            m = re.match(r"case (\w+) (\d+) B/rank n=(\d+): protocol (\d+) .* launches/device (\d+)", line)
            if m:
                cases += [(f"{m.group(1)} {int(m.group(2)) >> 20} MiB n={m.group(3)} proto {m.group(4)}",
                           int(m.group(5)))]
    names = []
    for name, k in cases:
        names += [f"{name} (warm-up)"] * (k - 1) + [name]
    print(f"{'launch':40s} {'us':>9s} {'tx MB':>9s} {'tx user':>9s} {'rx MB':>9s} {'rx user':>9s} "
          f"{'egress user GB/s':>17s} {'egress wire GB/s':>17s} {'wire/user':>9s}")
    for i in sorted(d):
        m = d[i]
        us = m["gpu__time_duration.sum"] / 1e3
        tx, txu = m["nvltx__bytes.sum"], m["nvltx__bytes_data_user.sum"]
        rx, rxu = m["nvlrx__bytes.sum"], m["nvlrx__bytes_data_user.sum"]
        name = names[i] if i < len(names) else m["kernel"][:40]
        print(f"{name:40s} {us:9.1f} {tx / 1e6:9.2f} {txu / 1e6:9.2f} {rx / 1e6:9.2f} {rxu / 1e6:9.2f} "
              f"{txu / us / 1e3:17.1f} {tx / us / 1e3:17.1f} {tx / max(txu, 1):9.3f}")


if __name__ == "__main__":
    main()
