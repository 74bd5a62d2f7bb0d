"""Time one feast_iterate against its pieces (projector, reduce) on a config: the rest is the
orthonormalisation, reduced eigenproblem (cuSOLVER) and Ritz vectors / residuals."""
import sys
import time

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


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return 1e3 * (time.perf_counter() - t0) / reps


Q = f.project(A, B, X)
tp = timed(lambda: f.project(A, B, X, Q))
tr = timed(lambda: f.reduce(A, B, Q))
Xi = X.clone()
ti = timed(lambda: f.iterate(A, B, Xi))
print(f"{key}: project {tp:.2f} ms, reduce {tr:.2f} ms, iterate {ti:.2f} ms -> rest {ti - tp - tr:.2f} ms")
