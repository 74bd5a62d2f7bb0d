"""Static SASS instruction counts per kernel of the built library (cuobjdump -sass): the FP64 tensor
(DMMA), operand staging (LDGSTS = cp.async, UTMALDG = TMA tensor load, UBLKCP = TMA bulk copy),
shared/global memory, distributed shared memory (STAS = st.async, SYNCS = mbarrier ops) and the
FP64 pipe (DFMA) instructions of each hot kernel.

    python tools/sass_counts.py [paper_1404_2891_b200/libfeast_b200.so] > profiles/r02/sass_counts.txt"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1404_2891_b200/libfeast_b200.so"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
OPS = ["DMMA", "DFMA", "LDGSTS", "UTMALDG", "UBLKCP", "LDS", "STS", "LDG", "STG", "STAS", "SYNCS", "REDUX", "SHFL",
       "BAR", "MUFU", "ATOMS"]
cur, counts = None, collections.OrderedDict()
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        counts[cur] = collections.Counter()
        continue
    m = re.search(r"/\*[0-9a-f]{4}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
    if cur and m and m.group(2) in OPS:
        counts[cur][m.group(2)] += 1
names = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout.splitlines()
print(f"# static SASS counts, {lib} (sm_100a); columns: " + " ".join(OPS))
for (mangled, c), d in zip(counts.items(), names):
    short = re.sub(r"\(.*", "", d.replace("(anonymous namespace)::", "").replace("feast::", "").replace("void ", ""))
    if any(k in short for k in ("zgemm", "panel", "trtri", "trsm", "laswp", "shift", "accum", "splitk", "gather",
                                "broadcast", "perm")):
        print(f"{short:72s} " + " ".join(f"{k}={c[k]}" for k in OPS if c[k]))
