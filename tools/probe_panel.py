"""Panel-kernel timing probe: per-launch panel time vs batch size and n (CUDA events)."""
import sys
import numpy as np, torch
sys.path.insert(0, '.')
import synth
from paper_1404_2891_b200 import Feast, feast as fb
for n, batch in [(2048, 1), (2048, 8), (2048, 16), (1024, 16), (512, 16)]:
    P = synth.make_pencil("C2", n=n, m0=128)
    s = P.spec
    f = Feast(P.n, P.m0, s.c, s.r, s.aspect, s.n_e, s.rule, fb.RIGHT, False, max_batch=batch)
    d = lambda a: torch.from_numpy(np.asfortranarray(a)).to("cuda")
    A, B, X = d(P.A), d(P.B), d(P.X0)
    Q = f.project(A, B, X)
    f.profile(True); f.project(A, B, X, Q); torch.cuda.synchronize()
    pr = f.profile_summary(); f.profile(False)
    p = pr["panel"]
    print(f"n={n} batch={batch}: panel {p['ms']:.2f} ms total, {1e3*p['ms']/p['launches']:.1f} us/launch "
          f"({1e3*p['ms']/p['launches']/64:.2f} us/col), zgemm {pr['zgemm']['ms']:.2f} ms", flush=True)
