"""Pins of oracle steps O2-O6: the right projector sum_j w_j (z_j B - A)^-1 (B X)
(eq. Rasp) and the left projector sum_j conj(w_j) (z_j B - A)^-H (B^H V)
(eq. Lasp, reading R4).

Pins independent of the oracle's arithmetic:
  * spectral identity rho(B^-1 A) = X rho(Lambda) Y^H B (eq. quadf_surM): on
    same-recipe shadows of C1, C2, C4, C5 (known V, lambda), Q* = V diag(rho(lambda)) V^-1 X
    with rho from the closed form 1/(1 + x^q) (numpy LAPACK solve for V^-1 X);
  * left identity (eq. quadf_surMconj): Q_L* = B^-H V^-H diag(conj rho) V^H B^H V_in;
  * S:263 worked example (golden file), U = 0 -> 0;
  * brute force with scipy.linalg.solve per node at n <= 64;
  * complex-symmetric invariant (B X)^T Q symmetric for the C3 recipe (C_j^T = C_j);
  * linearity; node-subset partition sums to the full sum (sharding, reading R17).
"""
import json
import os

import numpy as np
import pytest
import scipy.linalg as sla

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def _rho_closed(spec, lam):
    x = (lam - spec.c) / spec.r
    return 1.0 / (1.0 + x ** spec.q)


def test_spec_worked_example():
    g = json.load(open(os.path.join(GOLD, "filter_trapezoid_k3_unit_circle.json")))
    z, w = oracle.nodes(0.0, 1.0, 1.0, 4, 1)
    Q = oracle.project(np.diag([0.5, 3.0]).astype(complex), None, np.eye(2), z, w)
    want = np.diag([g["rho"][2][1], g["rho"][3][1]])
    assert np.max(np.abs(Q - want)) < 1e-7
    assert np.max(np.abs(Q - np.diag([1 / (1 - 0.5 ** 4), 1 / (1 - 3.0 ** 4)]))) < 1e-14
    assert np.array_equal(oracle.project(np.diag([0.5, 3.0]).astype(complex), None, np.zeros((2, 2)), z, w),
                          np.zeros((2, 2)))


@pytest.mark.parametrize("key,n,m0", [("C1", 200, 64), ("C2", 96, 24), ("C4", 128, 32), ("C5", 96, 32),
                                      ("R2", 96, 24)])
def test_spectral_identity_right(key, n, m0):
    P = synth.make_pencil(key, n=n, m0=m0)
    z, w = oracle.nodes(P.spec.c, P.spec.r, P.spec.aspect, P.spec.n_e, P.spec.rule)
    Q = oracle.project(P.A, P.B, P.X0, z, w)
    Qs = P.V @ (_rho_closed(P.spec, P.lam)[:, None] * np.linalg.solve(P.V, P.X0))
    assert _rel(Q, Qs) < 1e-11


@pytest.mark.parametrize("key,n,m0", [("C4", 128, 32), ("C2", 96, 24)])
def test_spectral_identity_left(key, n, m0):
    P = synth.make_pencil(key, n=n, m0=m0)
    z, w = oracle.nodes(P.spec.c, P.spec.r, P.spec.aspect, P.spec.n_e, P.spec.rule)
    Vin = synth.random_block(n, m0, 5)
    QL = oracle.project(P.A, P.B, Vin, z, w, left=True)
    Bm = np.eye(n) if P.B is None else P.B
    inner = P.V.conj().T @ (Bm.conj().T @ Vin)
    core = np.linalg.solve(P.V.conj().T, np.conj(_rho_closed(P.spec, P.lam))[:, None] * inner)
    QLs = np.linalg.solve(Bm.conj().T, core)
    assert _rel(QL, QLs) < 1e-11


@pytest.mark.parametrize("key", ["C1", "C2", "C3", "C4"])
@pytest.mark.parametrize("left", [False, True])
def test_brute_force_small(key, left):
    n, m0 = 48, 8
    P = synth.make_pencil(key, n=n, m0=m0)
    z, w = oracle.nodes(P.spec.c, P.spec.r, P.spec.aspect, P.spec.n_e, P.spec.rule)
    Bm = np.eye(n) if P.B is None else P.B
    ref = np.zeros((n, m0), complex)
    for zj, wj in zip(z, w):
        C = zj * Bm - P.A
        if left:
            ref += np.conj(wj) * sla.solve(C.conj().T, Bm.conj().T @ P.X0)
        else:
            ref += wj * sla.solve(C, Bm @ P.X0)
    assert _rel(oracle.project(P.A, P.B, P.X0, z, w, left=left), ref) < 1e-12


def test_complex_symmetric_invariant():
    P = synth.make_pencil("C3", n=160, m0=24)
    assert np.array_equal(P.A, P.A.T) and np.array_equal(P.B, P.B.T)
    z, w = oracle.nodes(P.spec.c, P.spec.r, P.spec.aspect, P.spec.n_e, P.spec.rule)
    Q = oracle.project(P.A, P.B, P.X0, z, w)
    M = (P.B @ P.X0).T @ Q
    assert np.linalg.norm(M - M.T) / np.linalg.norm(M) < 1e-12


def test_linearity_and_partition():
    P = synth.make_pencil("C2", n=64, m0=6)
    z, w = oracle.nodes(P.spec.c, P.spec.r, P.spec.aspect, P.spec.n_e, P.spec.rule)
    U1, U2 = synth.random_block(64, 6, 1), synth.random_block(64, 6, 2)
    al = 0.7 - 1.3j
    lhs = oracle.project(P.A, P.B, al * U1 + U2, z, w)
    rhs = al * oracle.project(P.A, P.B, U1, z, w) + oracle.project(P.A, P.B, U2, z, w)
    assert _rel(lhs, rhs) < 1e-12
    full = oracle.project(P.A, P.B, U1, z, w)
    for world in (2, 4, 8):
        parts = [oracle.project(P.A, P.B, U1, z, w, *synth.node_owner_range(len(z), r, world)) for r in range(world)]
        assert _rel(sum(parts), full) < 1e-13


def test_singular_node_detected():
    # a pole placed exactly on an eigenvalue: z_0 = 0.5 = lambda_0 of A = diag(0.5, 3)
    A = np.diag([0.5, 3.0]).astype(complex)
    z = np.array([0.5 + 0j, -1.0]); w = np.array([1.0 + 0j, 1.0])
    with pytest.raises(ZeroDivisionError):
        oracle.project(A, None, np.eye(2), z, w)


def test_real_pencil_conjugate_pole_symmetry():
    """Real pencil (R2 recipe) and a contour symmetric about the real axis: the partner pole's
    solve is the conjugate of the primary pole's solve with conj(R) (C(conj z) = conj(C(z))),
    the identity the real-pencil mode (NEXT-2b) relies on; checked with scipy solves."""
    P = synth.make_pencil("R2", n=40, m0=6)
    assert np.abs(P.A.imag).max() == 0.0 and np.abs(P.B.imag).max() == 0.0
    z, w = oracle.nodes(P.spec.c, P.spec.r, P.spec.aspect, P.spec.n_e, P.spec.rule)
    R = P.B @ P.X0
    for j, zj in enumerate(z):
        k = int(np.argmin(np.abs(z - np.conj(zj))))
        assert abs(z[k] - np.conj(zj)) < 1e-14 and abs(w[k] - np.conj(w[j])) < 1e-14
        Yk = sla.solve(z[k] * P.B - P.A, R)
        Yj_conj = np.conj(sla.solve(zj * P.B - P.A, np.conj(R)))
        assert _rel(Yj_conj, Yk) < 1e-12


@pytest.mark.parametrize("key", ["C1", "C2", "R2"])
def test_count_estimator_trace_identity(key):
    """NEXT-3 count estimate: tr(U^H rho(B^-1 A) U) with U = I equals tr rho(B^-1 A) =
    sum_i rho(lambda_i) (similarity invariance; rho from the closed form), and for random CN(0,1)
    U its expectation — checked here on the oracle projector at a small size."""
    P = synth.make_pencil(key, n=48, m0=48)
    z, w = oracle.nodes(P.spec.c, P.spec.r, P.spec.aspect, P.spec.n_e, P.spec.rule)
    Q = oracle.project(P.A, P.B, np.eye(P.n, dtype=complex), z, w)
    exact = np.sum(_rho_closed(P.spec, P.lam))
    assert abs(np.trace(Q) - exact) <= 1e-11 * max(1.0, abs(exact))
