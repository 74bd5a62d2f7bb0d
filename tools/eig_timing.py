import time, torch, numpy as np
for m in (64, 128, 256, 512):
    M = torch.randn(m, m, dtype=torch.complex128, device="cuda")
    for name, fn in [("eig", lambda: torch.linalg.eig(M)), ("eigvals", lambda: torch.linalg.eigvals(M))]:
        fn(); torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3): fn()
        torch.cuda.synchronize()
        print(m, name, f"{1e3*(time.perf_counter()-t0)/3:.2f} ms")
    Mh = M.cpu().numpy()
    t0 = time.perf_counter()
    for _ in range(3): np.linalg.eig(Mh)
    print(m, "numpy eig (host)", f"{1e3*(time.perf_counter()-t0)/3:.2f} ms")

import sys
sys.path.insert(0, ".")
from paper_1404_2891_b200 import feast as fb
for m in (64, 128, 160):
    M = torch.randn(m, m, dtype=torch.complex128, device="cuda")
    fb.small_eig(M); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3): fb.small_eig(M)
    torch.cuda.synchronize()
    print(m, "feast_small_eig (one CTA)", f"{1e3*(time.perf_counter()-t0)/3:.2f} ms")
