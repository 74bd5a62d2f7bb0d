"""One projection of a pivot-heavy pencil (the C3 recipe: random symmetric H + iD, partial pivoting
swaps in most columns) for ncu captures of the row-swap kernels (FEAST_LASWP selects the kernel).

    ncu --metrics ... -k regex:laswp python tools/swap_probe.py [n]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth
from paper_1404_2891_b200 import Feast, feast as fb

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
P = synth.make_pencil("C3", n=n, m0=64)
s = P.spec
f = Feast(P.n, P.m0, s.c, s.r, s.aspect, s.n_e, s.rule, fb.RIGHT, False, max_batch=8)
d = lambda a: torch.from_numpy(np.asfortranarray(a)).to("cuda")
A, B, X = d(P.A), d(P.B), d(P.X0)
Q = f.project(A, B, X)
f.profile(True, serial=True)
f.project(A, B, X, Q)
torch.cuda.synchronize()
p = f.profile_summary()["laswp"]
f.profile(False)
print(f"laswp: {p['launches']} launches, {p['ms']:.3f} ms, moved {p['bytes'] / 1e6:.1f} MB "
      f"-> {p['bytes'] / (p['ms'] * 1e-3) / 1e9 if p['ms'] else 0:.1f} GB/s (serialised, moved bytes only)")
