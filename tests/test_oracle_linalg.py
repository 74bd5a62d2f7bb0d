"""Pins of oracle steps O3/O4 (naive LU with partial pivoting, substitution, conj-transpose
solves) and O7 (reduced eigensolver).  Checked against textbook invariants and library
routines the oracle does not use: reconstruction P M = L U, residuals, scipy
solve of M^H, scipy.linalg.eig, diagonal examples."""
import numpy as np
import pytest
import scipy.linalg as sla

import oracle


def _rand(n, m, seed):
    r = np.random.default_rng(seed)
    return (r.standard_normal((n, m)) + 1j * r.standard_normal((n, m))) / np.sqrt(2)


def _unpack(LU, piv):
    n = LU.shape[0]
    L = np.tril(LU, -1) + np.eye(n)
    U = np.triu(LU)
    perm = np.arange(n)
    for k in range(n):
        perm[[k, piv[k]]] = perm[[piv[k], k]]
    return L, U, perm


def test_lu_trivial():
    LU, piv, info, _ = oracle.lu(np.eye(3))
    assert info == 0 and np.array_equal(LU, np.eye(3)) and list(piv) == [0, 1, 2]
    LU, piv, info, st = oracle.lu(np.diag([2, 4j]))
    assert np.allclose(LU, np.diag([2, 4j])) and list(piv) == [0, 1]
    assert st[0] == 2 and st[1] == 4


@pytest.mark.parametrize("n,seed", [(8, 0), (33, 1), (64, 2)])
def test_lu_reconstruction_and_pivot_rule(n, seed):
    M = _rand(n, n, seed)
    LU, piv, info, _ = oracle.lu(M)
    assert info == 0
    L, U, perm = _unpack(LU, piv)
    assert np.linalg.norm(M[perm] - L @ U) / np.linalg.norm(M) < 1e-13
    # partial pivoting on |re|+|im| (reading R7): |l_ij| <= |a|_1/|p|_1 * sqrt(2) <= sqrt(2)
    assert np.max(np.abs(L)) <= np.sqrt(2) + 1e-15
    assert sorted(perm) == list(range(n))


def test_lu_singular_flag():
    M = np.ones((4, 4), dtype=complex)
    _, _, info, st = oracle.lu(M)
    assert info != 0 and st[0] == 0.0


def test_solve_examples():
    LU, piv, _, _ = oracle.lu(np.diag([2, -1j]))
    x = oracle.lu_solve(LU, piv, np.array([2, -1j]))
    assert np.allclose(x[:, 0], [1, 1], atol=1e-15)


@pytest.mark.parametrize("n", [6, 20, 50])
def test_solve_direct_and_conjugate_transpose(n):
    M = _rand(n, n, n)
    Bm = _rand(n, 3, n + 1)
    LU, piv, _, _ = oracle.lu(M)
    X = oracle.lu_solve(LU, piv, Bm, 0)
    assert np.linalg.norm(M @ X - Bm) <= 1e-12 * np.linalg.norm(Bm) * np.linalg.cond(M)
    Xh = oracle.lu_solve(LU, piv, Bm, 2)
    ref = sla.solve(M.conj().T, Bm)
    assert np.linalg.norm(Xh - ref) / np.linalg.norm(ref) < 1e-10


def test_gemm_vs_numpy():
    Am, Bm = _rand(7, 5, 1), _rand(5, 4, 2)
    assert np.allclose(oracle.gemm(Am, Bm), Am @ Bm, atol=1e-14)
    Ah = _rand(5, 7, 3)
    assert np.allclose(oracle.gemm(Ah, Bm, opa=2), Ah.conj().T @ Bm, atol=1e-14)


def test_eig_spec_examples():
    lam, W = oracle.eig(np.diag([1.0, 2.0]), np.eye(2))
    assert np.allclose(np.sort_complex(lam), [1, 2])
    lam, W = oracle.eig(np.diag([1.0, 2.0]), 2 * np.eye(2))
    assert np.allclose(np.sort_complex(lam), [0.5, 1.0])


def _match(a, b):
    """max over a of distance to the nearest unused element of b (greedy one-to-one)."""
    b = list(b)
    worst = 0.0
    for x in sorted(a, key=lambda v: (v.real, v.imag)):
        d = [abs(x - y) for y in b]
        i = int(np.argmin(d))
        worst = max(worst, d[i])
        b.pop(i)
    return worst


@pytest.mark.parametrize("m,seed", [(5, 0), (16, 1), (40, 2), (64, 3)])
def test_eig_vs_scipy(m, seed):
    Ah = _rand(m, m, seed)
    Bh = np.eye(m) + 0.3 * _rand(m, m, seed + 100)
    lam, W = oracle.eig(Ah, Bh)
    ref = sla.eigvals(Ah, Bh)
    assert _match(lam, ref) < 1e-10 * max(1, np.max(np.abs(ref)))
    # eigenvector residuals and unit columns
    R = Ah @ W - (Bh @ W) * lam[None, :]
    assert np.max(np.linalg.norm(R, axis=0)) < 1e-11 * np.linalg.norm(Ah)
    assert np.allclose(np.linalg.norm(W, axis=0), 1.0)


def test_eig_permutation_similarity():
    m = 12
    Ah, Bh = _rand(m, m, 7), np.eye(m) + 0.2 * _rand(m, m, 8)
    P = np.eye(m)[np.random.default_rng(0).permutation(m)]
    l1, _ = oracle.eig(Ah, Bh)
    l2, _ = oracle.eig(P @ Ah @ P.T, P @ Bh @ P.T)
    assert _match(l1, l2) < 1e-10


def test_thread_count_does_not_change_results():
    """The oracle's OpenMP splits only independent work (nodes; a lone node's update columns and
    right-hand sides), so every result bit is the same for 1 thread and for all of them."""
    import os
    rng = np.random.default_rng(11)
    n = 640
    M = np.asfortranarray(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    R = np.asfortranarray(rng.standard_normal((n, 6)) + 1j * rng.standard_normal((n, 6)))
    z, w = oracle.nodes(0.1, 0.5, 1.0, 4, 0)
    out = []
    for t in (1, max(2, len(os.sched_getaffinity(0)))):
        oracle.threads(t)
        LU, piv, _, _ = oracle.lu(M)
        out.append((LU, oracle.lu_solve(LU, piv, R), oracle.gemm(M, R), oracle.project(M, M.T.copy(order="F"), R, z, w),
                    oracle.project(M, None, R, z, w, 1, 2, left=True)))
    for a, b in zip(*out):
        assert np.array_equal(a, b)
