"""Summarise a timeline CSV (tools/timeline.py --out): per-stream busy time, GEMM coverage of the
wall clock (time with at least one trailing-update GEMM running) and the gaps between them."""
import csv
import sys

R = list(csv.DictReader(open(sys.argv[1])))
for r in R:
    r["t0"], r["t1"], r["flops"] = float(r["t0"]), float(r["t1"]), float(r["flops"])
wall = max(r["t1"] for r in R)


def union(iv):
    iv = sorted(iv)
    tot, c0, c1 = 0.0, None, None
    for a, b in iv:
        if c1 is None or a > c1:
            if c1 is not None:
                tot += c1 - c0
            c0, c1 = a, b
        else:
            c1 = max(c1, b)
    return tot + ((c1 - c0) if c1 is not None else 0.0)


big = [(r["t0"], r["t1"]) for r in R if r["cls"] == "zgemm" and r["flops"] > 2e9]
anyk = [(r["t0"], r["t1"]) for r in R]
gemm_fl = sum(r["flops"] for r in R if r["cls"] == "zgemm")
print(f"wall {wall:.3f} ms; union of all kernels {union(anyk):.3f} ms; union of big GEMMs {union(big):.3f} ms")
print(f"GEMM flops {gemm_fl:.3e} -> {gemm_fl / (wall * 1e-3) / 1e12:.2f} TF/s over the wall")
for st in sorted(set(r["stream"] for r in R)):
    rs = [r for r in R if r["stream"] == st]
    print(f"  stream {st}: {len(rs)} launches, busy {union([(r['t0'], r['t1']) for r in rs]):.3f} ms")
