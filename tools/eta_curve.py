"""eta(r) of a rule on the reference circle ("eta(r) = min_t |rho(mu(r,t))| for r <= 1 - delta,
max_t |rho(mu(r,t))| for r >= 1 + delta", delta = 0.01), from the library's feast_filter (host code,
no GPU).  python tools/eta_curve.py [rule n_e aspect]   (rule: 0 midpoint, 1 endpoint, 2 GL)"""
import ctypes
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1404_2891_b200 import feast as fb

rule = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n_e = int(sys.argv[2]) if len(sys.argv) > 2 else 8
aspect = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
lib = fb.load_library()
h = ctypes.c_void_p()
assert lib.feast_init(ctypes.byref(h), 64, 8, 0.0, 0.0, 1.0, aspect, n_e, rule, 0, 1, 0, 1, 0, None) == 0
th = np.linspace(0, 2 * np.pi, 1024, endpoint=False)
print(f"rule {rule}, n_e {n_e}, aspect {aspect}")
for r in [0.0, 0.25, 0.5, 0.75, 0.9, 0.99, 1.01, 1.1, 1.25, 1.5, 2.0, 3.0, 4.0]:
    mu = (r * (np.cos(th) + 1j * aspect * np.sin(th))).astype(np.complex128)
    out = np.zeros_like(mu)
    lib.feast_filter(h, len(mu), mu.ctypes.data_as(ctypes.c_void_p), out.ctypes.data_as(ctypes.c_void_p))
    eta = np.min(np.abs(out)) if r < 1 else np.max(np.abs(out))
    print(f"  r = {r:4.2f}  eta = {eta:.6e}")
lib.feast_destroy(h)
