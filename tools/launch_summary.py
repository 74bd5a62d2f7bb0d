"""Summarise an ncu launch list (ncu --metrics gpu__time_duration.sum --csv --log-file F ...): per
kernel, launches, summed (cold-cache, serialised) duration and share.  The library's kernels are
grouped by name; everything else (torch fixture generation, cuSOLVER) is listed as well.

    python tools/launch_summary.py gpurun_out/r2_launches_C4.csv [--from-first feast_kernel_regex]"""
import collections
import csv
import re
import sys

path = sys.argv[1]
rows = [l for l in open(path) if l.startswith('"')]
R = list(csv.DictReader(rows))
start = 0
if "--from-first" in sys.argv:
    pat = re.compile(sys.argv[sys.argv.index("--from-first") + 1])
    start = next(i for i, r in enumerate(R) if pat.search(r["Kernel Name"]))
agg = collections.defaultdict(lambda: [0, 0.0])
SC = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}
for r in R[start:]:
    name = r["Kernel Name"]
    short = re.sub(r"^void ", "", name).replace("<unnamed>::", "").replace("(anonymous namespace)::", "").split("(")[0]
    short = re.sub(r"<.*", "", short).split("::")[-1]
    agg[short][0] += 1
    agg[short][1] += float(r["Metric Value"].replace(",", "")) * SC[r["Metric Unit"]]
tot = sum(v[1] for v in agg.values())
print(f"{len(R) - start} launches, {tot:.2f} ms summed kernel time")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]:
    print(f"{k:48s} {v[0]:6d} {v[1]:10.2f} ms {100 * v[1] / tot:5.1f}%")
