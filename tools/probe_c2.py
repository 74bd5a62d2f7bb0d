"""Quick timing probe of the projector on C2 (not the bench; CUDA events)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
import synth
from paper_1404_2891_b200 import Feast, feast as fb
key = sys.argv[1] if len(sys.argv) > 1 else "C2"
P = synth.make_pencil(key)
s = P.spec
f = Feast(P.n, P.m0, s.c, s.r, s.aspect, s.n_e, s.rule, fb.RIGHT, P.B is None)
d = lambda a: None if a is None else torch.from_numpy(np.asfortranarray(a)).to("cuda")
A, B, X = d(P.A), d(P.B), d(P.X0)
Q = f.project(A, B, X)
torch.cuda.synchronize()
for it in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); f.project(A, B, X, Q); e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1)
    n, m, q = P.n, P.m0, P.q
    fl = q * (8 / 3 * n ** 3 + 8 * n * n * m)
    print(f"{key} project {ms:.2f} ms  LU+solve {fl / ms / 1e9:.2f} TF/s  launches {f.last_launch_count}", flush=True)
f.profile(True)
f.project(A, B, X, Q)
torch.cuda.synchronize()
for k, v in f.profile_summary().items():
    if v["launches"]:
        extra = f"{v['flops'] / (v['ms'] * 1e-3) / 1e12:6.2f} TF/s" if v["flops"] else ""
        print(f"  {k:6s} n={v['launches']:4d} {v['ms']:8.3f} ms  {1e3 * v['ms'] / v['launches']:8.1f} us/launch {extra}")
f.profile(False)
