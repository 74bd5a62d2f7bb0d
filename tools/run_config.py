"""Run the projector (and reduce) on a full-size config on the GPU with property checks.

    python tools/run_config.py C3 [--batch 16] [--iters 1]
Prints timing and the checks: spectral identity Q = V rho(Lambda) V^-1 X (C1/C2/C4/C5, with the
closed-form filter and a cuSOLVER solve — independent of the FEAST kernels), the complex-
symmetric invariant (B X)^T Q symmetric (C3), left identity for bi configs."""
import argparse
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import synth
from paper_1404_2891_b200 import Feast, feast as fb

ap = argparse.ArgumentParser()
ap.add_argument("key")
ap.add_argument("--batch", type=int, default=0)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--m0", type=int, default=None)
ap.add_argument("--bi", action="store_true", help="force a Bi-FEAST handle (left + right blocks)")
ap.add_argument("--csym", action="store_true", help="complex-symmetric mode (NEXT-2a)")
ap.add_argument("--real", action="store_true", help="real-pencil mode (NEXT-2b)")
args = ap.parse_args()
t0 = time.time()
P = synth.make_pencil_torch(args.key, n=args.n, m0=args.m0)
torch.cuda.synchronize()
tgen = time.time() - t0
s = P.spec
bi = s.mode == "bi" or args.bi
f = Feast(P.n, P.m0, s.c, s.r, s.aspect, s.n_e, s.rule, fb.BI if bi else fb.RIGHT, P.B is None, max_batch=args.batch,
          complex_symmetric=args.csym, real_pencil=args.real)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
if bi:
    G = P.X0.conj().T @ P.X0
    V0 = torch.linalg.solve(G, P.X0.conj().T).conj().T.contiguous()   # X0 G^-H  (reading R6)
    V0 = V0.t().contiguous().t()
    e0.record(); Q, QL = f.project_bi(P.A, P.B, P.X0, V0); e1.record()
else:
    e0.record(); Q = f.project(P.A, P.B, P.X0); e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
n, m0, q = P.n, P.m0, P.q
fl = q * (8 / 3 * n ** 3 + 8 * n * n * m0 * (2 if bi else 1))
out = {"config": args.key, "n": n, "m0": m0, "q": q, "gen_s": round(tgen, 1), "project_ms": ms,
       "lu_solve_tflops": fl / (ms * 1e-3) / 1e12, "status": f.status}
if P.V is not None:
    x = (P.lam - s.c) / s.r
    rho = 1.0 / (1.0 + x ** q)
    Qs = P.V @ (rho[:, None] * torch.linalg.solve(P.V, P.X0))
    out["rel_err_spectral"] = float(torch.linalg.norm(Q - Qs) / torch.linalg.norm(Qs))
    if bi:
        inner = P.V.conj().T @ V0
        QLs = torch.linalg.solve(P.V.conj().T, rho.conj()[:, None] * inner)
        out["rel_err_spectral_left"] = float(torch.linalg.norm(QL - QLs) / torch.linalg.norm(QLs))
else:
    M = (P.B @ P.X0).T @ Q
    out["csym_asym"] = float(torch.linalg.norm(M - M.T) / torch.linalg.norm(M))
stats, worst = f.node_stats()
out["min_rel_pivot"] = min(v for v in stats if v >= 0)
print(json.dumps(out), flush=True)
