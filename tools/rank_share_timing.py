"""Per-rank compute time of a strong-scaled step (rank 0 of P owns q/P nodes): the projector of one
rank's node share + the (row-sharded) reduce, timed on one GPU — predicts the P-GPU step time
(the all-reduces over NVLink add ~n m0 16 B / 900 GB/s)."""
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
d = lambda a: None if a is None else torch.from_numpy(np.asfortranarray(a)).to("cuda")
A, B, X = d(P.A), d(P.B), d(P.X0)
base = None
for world in (1, 2, 4, 8):
    f = Feast(P.n, P.m0, s.c, s.r, s.aspect, s.n_e, s.rule, fb.RIGHT, P.B is None, rank=0, world=world, partial=True)
    Q = f.project(A, B, X)
    for _ in range(2):
        f.project(A, B, X, Q)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        f.project(A, B, X, Q)
        f.reduce(A, B, Q)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    base = base or ms
    print(f"{key} P={world}: rank share {ms:.3f} ms -> predicted efficiency {base / (world * ms):.2f}")
