"""Where a step's time goes, by phase: one serialised projector(+left) step (the roofline pass of
bench.py: one stream, CUDA events around every launch), split at the last panel launch into the
LU phase (shift, panels, swaps, triangular kernels, trailing updates incl. the fused forward
substitution) and the substitution phase (back substitution, left solves, accumulation); per
phase and class: time, algorithmic flops and TF/s.

    python tools/phase_breakdown.py C4 [--batch 0]"""
import argparse
import json
import sys
from collections import defaultdict

import torch

sys.path.insert(0, ".")
import synth
from paper_1404_2891_b200 import Feast, empty_colmajor, feast as fb

ap = argparse.ArgumentParser()
ap.add_argument("key", nargs="?", default="C4")
ap.add_argument("--batch", type=int, default=0)
ap.add_argument("--out", default=None)
args = ap.parse_args()
spec = synth.CONFIGS[args.key]
bi = spec.mode == "bi"
if spec.n >= 4096:
    P = synth.make_pencil_torch(args.key)
    A, B, X = P.A, P.B, P.X0
else:
    import numpy as np
    P = synth.make_pencil(args.key)
    d = lambda a: None if a is None else torch.from_numpy(np.asfortranarray(a)).to("cuda")
    A, B, X = d(P.A), d(P.B), d(P.X0)
n, m0 = P.n, P.m0
V = fb.colmajor(torch.linalg.solve(X.conj().T @ X, X.conj().T).conj().T) if bi else None
del P
torch.cuda.empty_cache()
f = Feast(n, m0, spec.c, spec.r, spec.aspect, spec.n_e, spec.rule, fb.BI if bi else fb.RIGHT, B is None,
          max_batch=args.batch)
Q = empty_colmajor(n, m0)
QL = empty_colmajor(n, m0) if bi else None


def step():
    if bi:
        f.project_bi(A, B, X, V, Q, QL)
    else:
        f.project(A, B, X, Q)


step()
f.profile(True, serial=True)
step()
torch.cuda.synchronize()
recs = f.profile_records()
f.profile(False)
last_panel = max(i for i, r in enumerate(recs) if r[0] == "panel")
out = {}
for name, sel in (("lu", recs[:last_panel + 1]), ("subst", recs[last_panel + 1:])):
    agg = defaultdict(lambda: [0, 0.0, 0.0])
    for c, st, t0, t1, fl in sel:
        a = agg[c]
        a[0] += 1
        a[1] += t1 - t0
        a[2] += fl
    out[name] = {c: {"launches": v[0], "ms": v[1], "tflops": (v[2] / (v[1] * 1e-3) / 1e12 if v[1] > 0 else None),
                     "flops": v[2]} for c, v in agg.items()}
    tot = sum(v[1] for v in agg.values())
    print(f"{args.key} {name}: {tot:.1f} ms")
    for c, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        tf = v[2] / (v[1] * 1e-3) / 1e12 if v[1] > 0 else 0
        print(f"   {c:6s} {v[0]:6d} launches {v[1]:10.2f} ms  {v[2]:.3e} flop  {tf:6.2f} TF/s")
if args.out:
    json.dump(out, open(args.out, "w"), indent=1)
# zgemm launches grouped by algorithmic flops per launch (one group = one launch shape)
by = defaultdict(lambda: [0, 0.0, 0.0])
for c, st, t0, t1, fl in recs:
    if c == "zgemm":
        g = by[round(fl, -3)]
        g[0] += 1
        g[1] += t1 - t0
        g[2] += fl
print("zgemm by launch shape (flops per launch): launches, ms, TF/s — top 25 by time")
for fl, v in sorted(by.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"   {fl:12.4e} flop/launch {v[0]:6d} launches {v[1]:9.3f} ms {v[2] / (v[1] * 1e-3) / 1e12:6.2f} TF/s")
# per phase: launch shapes ranked by time lost against the big trailing updates' rate
REF = 36.19   # TF/s of the C4 trailing updates (profiles/r02/phase_C4.txt)
for name, sel in (("lu", recs[:last_panel + 1]), ("subst", recs[last_panel + 1:])):
    byp = defaultdict(lambda: [0, 0.0, 0.0])
    for c, st, t0, t1, fl in sel:
        if c == "zgemm":
            g = byp[round(fl, -3)]
            g[0] += 1
            g[1] += t1 - t0
            g[2] += fl
    loss = {k: v[1] - v[2] / (REF * 1e9) for k, v in byp.items()}
    print(f"{name}: zgemm time lost vs {REF} TF/s: {sum(loss.values()):.2f} ms — top 20 shapes by loss")
    if args.out:
        out.setdefault("shapes", {})[name] = [[fl, v[0], v[1]] for fl, v in byp.items()]
        json.dump(out, open(args.out, "w"), indent=1)
    for fl, v in sorted(byp.items(), key=lambda kv: -loss[kv[0]])[:20]:
        print(f"   {fl:12.4e} flop/launch {v[0]:6d} launches {v[1]:9.3f} ms {v[2] / (v[1] * 1e-3) / 1e12:6.2f} TF/s"
              f"  lost {loss[fl]:8.2f} ms")
