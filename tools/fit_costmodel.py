"""Alpha-beta cost model of the PAT collectives, calibrated on the measured sweeps.

The reference prices a schedule as rounds x (alpha + beta x bytes) per topology level
(costmodel.cpp:70-104). On one NVSwitch box every peer is one hop away, so a single level
remains, and the protocol decides the constants:

    t(n, C) = a_p + b_p * R(n, T) + w_p * (n - 1) * C / B_p

R = PAT rounds (ceil(log2 n) at T = max_trees), C = chunk bytes, w_p = wire bytes per payload
byte (LL 2, LL32 32/28, SIMPLE 1), B_p = sustained link GB/s, a_p launch + completion, b_p per-round
synchronisation. Fitted by least squares on single-step points of forced-protocol sweeps.
Since (n-1)*C does not depend on T and b_p > 0, T = max_trees (fewest rounds) minimises t for
every size: the model justifies the library's fixed T. The LL/SIMPLE crossover it predicts is
compared with the library's threshold.

  python tools/fit_costmodel.py profiles/r01f_forced_n*_p{1,2}.jsonl profiles/r01f_ll32_noskew_n*.jsonl \
      > profiles/r01f_costmodel_fit.json
"""
import argparse
import json
import math

import numpy as np

WIRE = {1: 2.0, 2: 1.0, 5: 32.0 / 28.0}  # protocol -> wire bytes per payload byte
NAME = {1: "LL", 2: "SIMPLE", 5: "LL32"}
STEP_BYTES = {"LL": 32 * 16 * 1024, "LL32": 148 * 28 * 1024}  # one polling step: channels x slot payload (LL: 32-channel region)


def rounds(n):
    return max(1, math.ceil(math.log2(n))) if n > 1 else 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("files", nargs="+")
    ap.add_argument("--out", default=None)
    ap.add_argument("--ll-threshold", type=int, default=2 << 20)
    args = ap.parse_args()
    pts = {1: [], 2: [], 5: []}
    for f in args.files:
        for line in open(f):
            r = json.loads(line)
            if r.get("impl") != "pat":
                continue
            p = r["plan"]["protocol"]
            if p not in pts or (r["plan"]["iterations"] != 1 and p != 5):
                continue  # LL and SIMPLE: single-step points; LL32's extra steps cost nothing (library model)
            n, C = r["n"], r["bytes_per_rank"]
            pts[p].append((n, C, r["us"]))
    fit = {}
    for p, v in pts.items():
        if len(v) < 3:
            continue
        X = np.array([[1.0, rounds(n), WIRE[p] * (n - 1) * C / 1e3] for n, C, _ in v])  # MB-ish units -> us
        y = np.array([t for _, _, t in v])
        coef, *_ = np.linalg.lstsq(X, y, rcond=None)
        a, b, inv = coef
        pred = X @ coef
        fit[NAME[p]] = {"a_us": float(a), "b_us_per_round": float(b), "link_gbs": float(1.0 / inv) if inv > 0 else None,
                        "wire": WIRE[p], "points": len(v),
                        "rel_err_median": float(np.median(np.abs(pred - y) / y)),
                        "rel_err_max": float(np.max(np.abs(pred - y) / y))}
    out = {"model": "t = a + b*R + w*(n-1)*C/B", "fit": fit, "crossover_bytes": {}}
    for ll in ("LL", "LL32"):
        if ll not in fit or "SIMPLE" not in fit:
            continue
        L, S = fit[ll], fit["SIMPLE"]
        out["crossover_bytes"][ll] = {}
        for n in range(2, 9):
            R = rounds(n)
            # a polling protocol beyond one step pays its fixed cost again per extra step
            best = None
            for k in range(10, 28):
                C = 1 << k
                steps = max(1, -(-C // STEP_BYTES[ll])) if ll == "LL" else 1
                tl = steps * (L["a_us"] + L["b_us_per_round"] * R) + L["wire"] * (n - 1) * C / (L["link_gbs"] * 1e3)
                ts = S["a_us"] + S["b_us_per_round"] * R + S["wire"] * (n - 1) * C / (S["link_gbs"] * 1e3)
                if tl > ts:
                    best = C
                    break
            out["crossover_bytes"][ll][n] = best
    out["library_ll_threshold"] = args.ll_threshold
    print(json.dumps(out, indent=1))
    if args.out:
        with open(args.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
