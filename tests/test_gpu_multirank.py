"""The real multi-rank data plane (the q linear systems distributed over processes) on
ONE GPU: two processes, a torch.distributed process group (gloo backend on CUDA tensors), each
rank a Feast handle with world = 2 whose library calls the registered all-reduce callback for the
node sum of Q / QL (a6), the row-sharded R = B X (a1) and A Q / B Q (a7), and the residual norms
of feast_iterate.  Every rank must return the FULL results, equal to the oracle's.

(The ranks' kernels never wait on each other: each rank runs its own nodes and only the
collectives synchronise, through gloo's host copies — so sharing one GPU is safe.)"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
TOL = 1e-10


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import torch.distributed as dist

    import synth
    from gpu_util import dev, host
    from paper_1404_2891_b200 import Feast, feast as fb
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = {}
    # C2 shadow (B != I): a1 sharded, node sum, a7 sharded
    P = synth.make_pencil("C2", n=260, m0=20)
    s = P.spec
    f = Feast(P.n, P.m0, s.c, s.r, s.aspect, s.n_e, s.rule, fb.RIGHT, False, rank=rank, world=world)
    A, B, X = dev(P.A), dev(P.B), dev(P.X0)
    Q = f.project(A, B, X)
    Ah, Bh = f.reduce(A, B, Q)
    res["c2_Q"], res["c2_Ah"], res["c2_Bh"] = host(Q), host(Ah), host(Bh)
    # a caller ld != n (the library packs the block for the collective)
    Qbig = torch.zeros((P.m0, P.n + 7), dtype=torch.complex128, device="cuda").t()
    f.project(A, B, X, Qbig[:P.n])
    res["c2_Q_ld"] = host(Qbig[:P.n])
    # C4 shadow, Bi-FEAST: Q and QL in one collective
    P4 = synth.make_pencil("C4", n=300, m0=24)
    s4 = P4.spec
    g = Feast(P4.n, P4.m0, s4.c, s4.r, s4.aspect, s4.n_e, s4.rule, fb.BI, True, rank=rank, world=world)
    V0 = P4.X0 @ np.linalg.inv(P4.X0.conj().T @ P4.X0).conj().T
    Q4, QL4 = g.project_bi(dev(P4.A), None, dev(P4.X0), dev(V0))
    res["c4_Q"], res["c4_QL"] = host(Q4), host(QL4)
    # C1: ten R-FEAST iterations (projector, node sum, sharded a7, sharded residuals)
    P1 = synth.make_pencil("C1")
    s1 = P1.spec
    h = Feast(P1.n, P1.m0, s1.c, s1.r, s1.aspect, s1.n_e, s1.rule, fb.RIGHT, True, rank=rank, world=world)
    A1, X1 = dev(P1.A), dev(P1.X0)
    for _ in range(s1.iters):
        out = h.iterate(A1, None, X1)
    res["c1_lam"] = np.asarray(out["lam"])
    res["c1_resid"] = np.asarray(out["resid"])
    res["c1_flags"] = np.asarray(out["flags"])
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), **res)
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_one_gpu_full_results(tmp_path):
    import oracle
    import synth
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    P = synth.make_pencil("C2", n=260, m0=20)
    s = P.spec
    z, w = oracle.nodes(s.c, s.r, s.aspect, s.n_e, s.rule)
    Qo = oracle.project(P.A, P.B, P.X0, z, w)
    Aho = oracle.gemm(Qo, oracle.gemm(P.A, Qo), opa=2)
    Bho = oracle.gemm(Qo, oracle.gemm(P.B, Qo), opa=2)
    P4 = synth.make_pencil("C4", n=300, m0=24)
    s4 = P4.spec
    z4, w4 = oracle.nodes(s4.c, s4.r, s4.aspect, s4.n_e, s4.rule)
    V0 = P4.X0 @ np.linalg.inv(P4.X0.conj().T @ P4.X0).conj().T
    Q4o = oracle.project(P4.A, None, P4.X0, z4, w4)
    QL4o = oracle.project(P4.A, None, V0, z4, w4, left=True)
    P1 = synth.make_pencil("C1")
    s1 = P1.spec
    inside = P1.lam[np.abs(P1.lam - s1.c) < s1.r]
    rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
    lams = []
    for r in range(world):
        d = np.load(tmp_path / f"rank{r}.npz")
        assert rel(d["c2_Q"], Qo) <= TOL and rel(d["c2_Q_ld"], Qo) <= TOL
        assert rel(d["c2_Ah"], Aho) <= 1e-10 and rel(d["c2_Bh"], Bho) <= 1e-10
        assert rel(d["c4_Q"], Q4o) <= TOL and rel(d["c4_QL"], QL4o) <= TOL
        conv = (d["c1_flags"] & 1).astype(bool) & (d["c1_resid"] <= 1e-10)
        got = d["c1_lam"][conv]
        assert len(got) >= 1
        for x in got:                        # each converged Ritz value is a true eigenvalue
            assert np.min(np.abs(inside - x)) <= 1e-10 * s1.r
        lams.append(np.sort_complex(got))
    assert len(lams[0]) == len(lams[1]) and np.max(np.abs(lams[0] - lams[1])) <= 1e-12


def _nccl_worker(rank, port, outdir):
    """ONE process, an NCCL process group of size 1 (NCCL cannot put two ranks on one GPU), and
    two handles that each believe world = 2 (ranks 0 and 1): every node sum then goes through the
    real NCCL all-reduce on the library's raw staging block and stream (identity for one rank), so
    each handle returns its own ranks' partial sum, and the two partials add up to the full Q."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import torch.distributed as dist

    import synth
    from gpu_util import dev, host
    from paper_1404_2891_b200 import Feast, feast as fb
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    res = {}
    P4 = synth.make_pencil("C4", n=300, m0=24)   # B = I: no row-sharded a1 (identity sum would drop rows)
    s4 = P4.spec
    V0 = P4.X0 @ np.linalg.inv(P4.X0.conj().T @ P4.X0).conj().T
    A, X, V = dev(P4.A), dev(P4.X0), dev(V0)
    for r in range(2):
        g = Feast(P4.n, P4.m0, s4.c, s4.r, s4.aspect, s4.n_e, s4.rule, fb.BI, True, rank=r, world=2, partial=True)
        assert g.lib.feast_set_partial(g.h, 0) == 0          # full node sums, through NCCL:
        g._ar = fb.ALLREDUCE_FN(fb.make_allreduce_callback(g.device))
        assert g.lib.feast_set_allreduce(g.h, g._ar, None) == 0
        for call in range(3):                      # eager, captured, replayed graph
            Q, QL = g.project_bi(A, None, X, V)
            res[f"Q{r}_{call}"], res[f"QL{r}_{call}"] = host(Q), host(QL)
    np.savez(os.path.join(outdir, "nccl.npz"), **res)
    dist.destroy_process_group()


def test_nccl_allreduce_callback_partials(tmp_path):
    """The node sum through the binding's callback on the NCCL backend (the multi-GPU bench's
    collective): each world = 2 handle's result equals the oracle's sum over that rank's nodes
    (R17: rank r owns [r q/2, (r+1) q/2)), unchanged across graph capture and replay; the two
    partials add up to the oracle's Q / Q_L."""
    import oracle
    import synth
    mp.spawn(_nccl_worker, args=(_free_port(), str(tmp_path)), nprocs=1, join=True)
    d = np.load(tmp_path / "nccl.npz")
    P4 = synth.make_pencil("C4", n=300, m0=24)
    s4 = P4.spec
    z, w = oracle.nodes(s4.c, s4.r, s4.aspect, s4.n_e, s4.rule)
    V0 = P4.X0 @ np.linalg.inv(P4.X0.conj().T @ P4.X0).conj().T
    q = len(z)
    rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
    for r in range(2):
        j0, j1 = r * q // 2, (r + 1) * q // 2
        Qo = oracle.project(P4.A, None, P4.X0, z, w, j0, j1)
        QLo = oracle.project(P4.A, None, V0, z, w, j0, j1, left=True)
        for call in range(3):
            assert rel(d[f"Q{r}_{call}"], Qo) <= TOL and rel(d[f"QL{r}_{call}"], QLo) <= TOL
    Qfull = oracle.project(P4.A, None, P4.X0, z, w)
    assert rel(d["Q0_2"] + d["Q1_2"], Qfull) <= TOL
