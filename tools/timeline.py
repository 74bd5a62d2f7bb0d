"""Per-launch timeline of one projector call (CUDA events around every launch, both streams).

    python tools/timeline.py [C2] [--out gpurun_out/timeline_C2.csv]
Prints the wall time, per-stream busy time and idle gaps; writes class,stream,t0,t1,flops rows."""
import argparse
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth
from paper_1404_2891_b200 import Feast, feast as fb

ap = argparse.ArgumentParser()
ap.add_argument("key", nargs="?", default="C2")
ap.add_argument("--out", default=None)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--batch", type=int, default=0)
ap.add_argument("--world", type=int, default=1, help="time rank 0's node share of a P-rank job")
args = ap.parse_args()
spec = synth.CONFIGS[args.key]
bi = spec.mode == "bi"
if (args.n or spec.n) >= 4096:
    P = synth.make_pencil_torch(args.key, n=args.n)
    A, B, X = P.A, P.B, P.X0
else:
    P = synth.make_pencil(args.key, n=args.n)
    d = lambda a: None if a is None else torch.from_numpy(np.asfortranarray(a)).to("cuda")
    A, B, X = d(P.A), d(P.B), d(P.X0)
s = P.spec
V = fb.colmajor(torch.linalg.solve(X.conj().T @ X, X.conj().T).conj().T) if bi else None
n, m0 = P.n, P.m0
del P
torch.cuda.empty_cache()
f = Feast(n, m0, s.c, s.r, s.aspect, s.n_e, s.rule, fb.BI if bi else fb.RIGHT, B is None, max_batch=args.batch,
          world=args.world, partial=args.world > 1)
Q = fb.empty_colmajor(n, m0)
QL = fb.empty_colmajor(n, m0) if bi else None


def proj():
    if bi:
        f.project_bi(A, B, X, V, Q, QL)
    else:
        f.project(A, B, X, Q)


proj()
proj()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(f.stream)
proj()
e1.record(f.stream)
torch.cuda.synchronize()
print(f"{args.key}: project without events {e0.elapsed_time(e1):.3f} ms")
f.profile(True)
proj()
recs = f.profile_records()
f.profile(False)
wall = max(r[3] for r in recs)
print(f"with events: wall {wall:.3f} ms, {len(recs)} launches")
for st in (0, 1):
    busy = sum(r[3] - r[2] for r in recs if r[1] == st)
    print(f"  stream {st}: busy {busy:.3f} ms")
# union of busy intervals and idle gaps
iv = sorted((r[2], r[3]) for r in recs)
union, gaps, cur0, cur1 = 0.0, [], iv[0][0], iv[0][1]
for a, b in iv[1:]:
    if a > cur1:
        union += cur1 - cur0
        gaps.append((cur1, a - cur1))
        cur0, cur1 = a, b
    else:
        cur1 = max(cur1, b)
union += cur1 - cur0
print(f"  union busy {union:.3f} ms, idle {wall - union:.3f} ms in {len(gaps)} gaps")
bycls = {}
for c, st, a, b, fl in recs:
    k = (c, st)
    bycls.setdefault(k, [0, 0.0, 0.0])
    bycls[k][0] += 1
    bycls[k][1] += b - a
    bycls[k][2] += fl
for (c, st), (nl, ms, fl) in sorted(bycls.items(), key=lambda kv: -kv[1][1]):
    tf = f"{fl / (ms * 1e-3) / 1e12:6.2f} TF/s" if fl and ms > 0 else ""
    print(f"  {c:6s} s{st} {nl:5d} launches {ms:8.3f} ms {tf}")
if args.out:
    with open(args.out, "w") as fh:
        fh.write("cls,stream,t0,t1,flops\n")
        for r in recs:
            fh.write(f"{r[0]},{r[1]},{r[2]:.6f},{r[3]:.6f},{r[4]:.6g}\n")
