"""Pins of oracle steps O7-O9 (Rayleigh–Ritz, one R-FEAST / Bi-FEAST iteration, residuals
and flags).

  * Rayleigh–Ritz exactness on the full space: m0 = n, one iteration returns the
    full spectrum (vs scipy.linalg.eigvals(A, B)).
  * C1 (full BASELINE size, n = 200): after 10 R-FEAST iterations the converged inside
    Ritz values (resid <= 1e-10) equal eigenvalues lambda_i known by construction.
  * Bi-FEAST on a C4-recipe shadow: biorthogonality V^H B X = I and converged
    Ritz values equal the known lambda_i; Bi reaches at least as many converged pairs.
"""
import numpy as np
import pytest
import scipy.linalg as sla

import oracle
import synth


def _nearest(lam, truth):
    return np.array([np.min(np.abs(truth - l)) for l in lam])


def test_full_space_exactness():
    n = 12
    P = synth.make_pencil("C2", n=n, m0=n)
    # contour enclosing the whole spectrum so rho(B^-1 A) is well conditioned
    c, R = 0.0, 1.6
    z, w = oracle.nodes(c, R, 1.0, 32, 0)
    out = oracle.feast_iterate(P.A, P.B, P.X0, None, z, w, c, R, 1.0)
    ref = sla.eigvals(P.A, P.B)
    assert np.max(_nearest(out["lam"], ref)) < 1e-10
    assert np.max(out["resid"]) < 1e-12


def test_c1_rfeast_converges_to_known_eigenvalues():
    P = synth.make_pencil("C1")
    s = P.spec
    z, w = oracle.nodes(s.c, s.r, s.aspect, s.n_e, s.rule)
    X = P.X0
    for _ in range(s.iters):
        out = oracle.feast_iterate(P.A, P.B, X, None, z, w, s.c, s.r, s.aspect)
        X = out["X"]
    conv = (out["flags"] & 1).astype(bool) & (out["resid"] <= 1e-10)
    assert conv.sum() >= 1
    inside_true = np.abs(P.lam - s.c) < s.r
    assert conv.sum() <= inside_true.sum()
    err = _nearest(out["lam"][conv], P.lam[inside_true])
    assert np.max(err) <= 1e-10 * max(1.0, s.r)
    # Ritz vectors have unit 2-norm (reading R14)
    assert np.allclose(np.linalg.norm(X, axis=0), 1.0)


def test_bifeast_shadow():
    n, m0 = 160, 24
    P = synth.make_pencil("C4", n=n, m0=m0)
    s = P.spec
    z, w = oracle.nodes(s.c, s.r, s.aspect, s.n_e, s.rule)
    X = P.X0
    G = X.conj().T @ X
    V = X @ np.linalg.inv(G).conj().T          # reading R6: V0 = X0 G^-H, G = X0^H B X0
    assert np.allclose(V.conj().T @ X, np.eye(m0), atol=1e-12)
    for _ in range(4):
        out = oracle.feast_iterate(P.A, P.B, X, V, z, w, s.c, s.r, s.aspect)
        X, V = out["X"], out["V"]
    assert np.linalg.norm(V.conj().T @ X - np.eye(m0)) < 1e-8
    conv = (out["flags"] & 1).astype(bool) & (out["resid"] <= 1e-10)
    inside_true = np.abs(P.lam - s.c) < s.r
    assert conv.sum() == inside_true.sum() >= 1
    assert np.max(_nearest(out["lam"][conv], P.lam[inside_true])) <= 1e-10 * s.r
