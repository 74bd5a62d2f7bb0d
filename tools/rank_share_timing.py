"""Per-rank compute time of a strong-scaled step (rank 0 of P owns q/P nodes): the projector(s) of
one rank's node share + the row-sharded a1 / a7, timed on one GPU (a no-op all-reduce callback
stands in for the collectives, so the library takes its sharded paths) — predicts the P-GPU step
time.  The collectives it leaves out: one all-reduce of n m0 (x2 Bi) complex128 (the node sum)
and the m0 x m0 partials; over NVLink 5 (~900 GB/s per direction) the node sum of C4 (268 MB)
takes ~0.6 ms against a step of seconds.

    python tools/rank_share_timing.py C4 [--worlds 1,2,4,8] [--steps 2]"""
import argparse
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth
from paper_1404_2891_b200 import Feast, empty_colmajor, feast as fb

ap = argparse.ArgumentParser()
ap.add_argument("key", nargs="?", default="C2")
ap.add_argument("--worlds", default="1,2,4,8")
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--out", default=None)
args = ap.parse_args()
spec = synth.CONFIGS[args.key]
bi = spec.mode == "bi"
if spec.n >= 4096:
    P = synth.make_pencil_torch(args.key)
    A, B, X = P.A, P.B, P.X0
else:
    P = synth.make_pencil(args.key)
    d = lambda a: None if a is None else torch.from_numpy(np.asfortranarray(a)).to("cuda")
    A, B, X = d(P.A), d(P.B), d(P.X0)
n, m0 = P.n, P.m0
V = fb.colmajor(torch.linalg.solve(X.conj().T @ X, X.conj().T).conj().T) if bi else None
del P
torch.cuda.empty_cache()
noop = fb.ALLREDUCE_FN(lambda buf, count, stream, user: 0)
res = []
base = None
for world in [int(x) for x in args.worlds.split(",")]:
    f = Feast(n, m0, spec.c, spec.r, spec.aspect, spec.n_e, spec.rule, fb.BI if bi else fb.RIGHT, B is None,
              rank=0, world=world, partial=True)
    if world > 1:
        f.lib.feast_set_allreduce(f.h, noop, None)   # sharded a1 / a7 (partial: no node sum)
    Q = empty_colmajor(n, m0)
    QL = empty_colmajor(n, m0) if bi else None

    def step():
        if bi:
            f.project_bi(A, B, X, V, Q, QL)
        else:
            f.project(A, B, X, Q)
        f.reduce(A, B, Q, QL)

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(f.stream)
    for _ in range(args.steps):
        step()
    e1.record(f.stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    base = base or ms
    comm_ms = (1 + bi) * n * m0 * 16 * 2 * (world - 1) / world / 900e9 * 1e3 if world > 1 else 0.0
    eff = base / (world * (ms + comm_ms))
    res.append({"config": args.key, "P": world, "nodes_per_rank": spec.q // world, "rank_share_ms": ms,
                "allreduce_ms_est": comm_ms, "predicted_efficiency": eff})
    print(f"{args.key} P={world}: rank share {ms:.3f} ms (+ all-reduce ~{comm_ms:.2f} ms) -> predicted "
          f"efficiency {eff:.3f}", flush=True)
    del f
    torch.cuda.empty_cache()
if args.out:
    json.dump(res, open(args.out, "w"), indent=1)
