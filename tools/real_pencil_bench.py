"""Real-pencil mode (NEXT-2b) vs per-node factorisation on the R2 companion recipe: projector
time (CUDA events, steady state: graph replay) and LU+solve TF/s of the per-node algorithm."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth
from paper_1404_2891_b200 import Feast, feast as fb

P = synth.make_pencil("R2", n=int(sys.argv[1]) if len(sys.argv) > 1 else None)
s = P.spec
d = lambda a: torch.from_numpy(np.asfortranarray(a)).to("cuda")
A, B, X = d(P.A), d(P.B), d(P.X0)
out = {}
for real in (False, True):
    f = Feast(P.n, P.m0, s.c, s.r, s.aspect, s.n_e, s.rule, fb.RIGHT, False, real_pencil=real)
    Q = f.project(A, B, X)
    for _ in range(2):
        f.project(A, B, X, Q)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        f.project(A, B, X, Q)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    out[real] = (ms, Q.clone())
    n, m, q = P.n, P.m0, P.q
    fl = q * (8 / 3 * n ** 3 + 8 * n * n * m)
    print(f"R2 n={n} real_pencil={real}: project {ms:.3f} ms  (per-node-equivalent LU+solve {fl / ms / 1e9:.2f} TF/s)")
print(f"speedup {out[False][0] / out[True][0]:.2f}x, rel diff {float(torch.linalg.norm(out[True][1] - out[False][1]) / torch.linalg.norm(out[False][1])):.2e}")
