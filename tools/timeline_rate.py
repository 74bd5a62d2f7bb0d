"""FLOP rate over time from a timeline CSV (tools/timeline.py --out): the wall clock cut into
bins, each launch's flops spread evenly over its [t0, t1]; prints TF/s per bin and which kernel
classes were running, to show where the machine idles (start-up, the LU tail, the solves).

    python tools/timeline_rate.py gpurun_out/timeline_C3.csv [bins]"""
import csv
import sys
from collections import defaultdict

R = list(csv.DictReader(open(sys.argv[1])))
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for r in R:
    r["t0"], r["t1"], r["flops"] = float(r["t0"]), float(r["t1"]), float(r["flops"])
wall = max(r["t1"] for r in R)
w = wall / nb
rate = [0.0] * nb
busy = [defaultdict(float) for _ in range(nb)]
for r in R:
    d = max(r["t1"] - r["t0"], 1e-9)
    b0, b1 = int(r["t0"] / w), min(int(r["t1"] / w), nb - 1)
    for b in range(b0, b1 + 1):
        lo, hi = max(r["t0"], b * w), min(r["t1"], (b + 1) * w)
        if hi > lo:
            rate[b] += r["flops"] * (hi - lo) / d
            busy[b][r["cls"]] += hi - lo
tot = sum(r["flops"] for r in R)
print(f"wall {wall:.3f} ms, {tot:.3e} flop, {tot / wall / 1e9:.2f} TF/s average")
for b in range(nb):
    tf = rate[b] / w / 1e9
    cl = ", ".join(f"{k} {v / w:.1f}" for k, v in sorted(busy[b].items(), key=lambda x: -x[1]) if v / w >= 0.05)
    print(f"{b * w:9.2f}-{(b + 1) * w:9.2f} ms {tf:6.2f} TF/s {'#' * int(tf)}  [{cl}]")
