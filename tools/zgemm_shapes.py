"""Where the dominant kernel loses its FP64 rate: one serialised C2 bench step (the roofline pass
of bench.py), zgemm launches grouped by algorithmic flops (= shape), with time and TF/s.

    python tools/zgemm_shapes.py [C2]"""
import sys
from collections import defaultdict

import numpy as np
import torch

sys.path.insert(0, ".")
import synth
from paper_1404_2891_b200 import Feast, feast as fb

key = sys.argv[1] if len(sys.argv) > 1 else "C2"
P = synth.make_pencil(key)
s = P.spec
f = Feast(P.n, P.m0, s.c, s.r, s.aspect, s.n_e, s.rule, fb.RIGHT, P.B is None)
d = lambda a: None if a is None else torch.from_numpy(np.asfortranarray(a)).to("cuda")
A, B, X = d(P.A), d(P.B), d(P.X0)
Q = torch.empty_like(X)
for it in range(3):
    f.profile(True, serial=True)
    f.project(A, B, X, Q)
    torch.cuda.synchronize()
recs = f.profile_records()
f.profile(False)
by = defaultdict(lambda: [0, 0.0, 0.0])
cls_ms = defaultdict(float)
for c, st, t0, t1, fl in recs:
    cls_ms[c] += t1 - t0
    if c != "zgemm":
        continue
    b = by[round(fl / 1e6, 1)]
    b[0] += 1
    b[1] += t1 - t0
    b[2] += fl
tot = sum(v[1] for v in by.values())
print(f"{key}: serialised project {sum(cls_ms.values()):.3f} ms; per class " +
      ", ".join(f"{k} {v:.3f}" for k, v in sorted(cls_ms.items(), key=lambda x: -x[1])))
print(f"zgemm {tot:.3f} ms, {sum(v[2] for v in by.values()) / tot / 1e9:.2f} TF/s")
print(f"{'MFLOP/launch':>14} {'count':>6} {'ms':>8} {'share':>6} {'TF/s':>7} {'lost_ms@37':>10}")
rows = sorted(by.items(), key=lambda kv: -(kv[1][1] - kv[1][2] / 37.17e9))
for k, (c, ms, fl) in rows[:40]:
    print(f"{k:14.1f} {c:6d} {ms:8.3f} {ms / tot:6.3f} {fl / ms / 1e9:7.2f} {ms - fl / 37.17e9:10.3f}")
