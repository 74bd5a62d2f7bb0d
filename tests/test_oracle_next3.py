"""Pins of the oracle's NEXT-3 functions: the eigenvalue-count estimate from
eig(V^^H B U^), the candidate monitors Res_(k) / trace_(k) and the
filter-gap report.

  * full space (p = n, V^H B U = I): V^^H B U^ = U^-1 rho(B^-1 A)^2 U, so its eigenvalues are
    rho(lambda_i)^2 exactly — lambda_i known by construction, rho from the closed form
    1/(1 + x^q) (reading R1): binds both projectors (left weights conjugated) and the product;
  * eigenvector subspace (U = right, V = left eigenvectors with V^H B U = I): V^^H B U^ =
    diag(rho(lambda_S)^2);
  * counts: a pencil with 3 eigenvalues deep inside and the rest far outside counts 3;
  * Bi-FEAST on a C4-recipe shadow: trace_(k) = the sum of the known inside eigenvalues once all
    have converged, Res_(k) small; the count estimate at the last iterate equals m;
  * filter gap: circle examples whose |rho| = 1/|1 + x^q| is a closed form, including an outside
    eigenvalue whose |rho| exceeds an inside one (m' > m)."""
import numpy as np
import pytest

import oracle
import synth


def _rho_closed(P, lam):
    s = P.spec
    return 1.0 / (1.0 + ((lam - s.c) / s.r) ** s.q)


def _bi_start(P, U):
    G = U.conj().T @ (U if P.B is None else P.B @ U)
    return U @ np.linalg.inv(G).conj().T          # reading R6: V^H B U = I


@pytest.mark.parametrize("key", ["C1", "C2", "C4"])
def test_full_space_eigs_are_rho_squared(key):
    n = 24
    P = synth.make_pencil(key, n=n, m0=n)
    s = P.spec
    z, w = oracle.nodes(s.c, s.r, s.aspect, s.n_e, s.rule)
    U = P.X0
    mu = oracle.bhat_eigs(P.A, P.B, U, _bi_start(P, U), z, w)
    ref = list(_rho_closed(P, P.lam) ** 2)
    assert np.all(np.diff(np.abs(mu)) <= 0)                  # sorted by decreasing modulus
    for x in mu:                                             # one-to-one nearest match
        d = np.abs(np.asarray(ref) - x)
        i = int(np.argmin(d))
        assert d[i] <= 1e-10 * max(1.0, abs(x)), (x, ref[i])
        ref.pop(i)


def test_eigenvector_subspace_gives_diagonal():
    """U = V_S (right eigenvectors of B^-1 A = V Lambda V^-1), V = (B^-H V^-H)_S (left ones),
    V^H B U = I: V^^H B U^ = diag(rho(lambda_S)^2) exactly."""
    n = 40
    P = synth.make_pencil("C2", n=n, m0=6)
    s = P.spec
    z, w = oracle.nodes(s.c, s.r, s.aspect, s.n_e, s.rule)
    r = np.abs(_rho_closed(P, P.lam))
    S = np.argsort(-r)[:6]
    U = np.asfortranarray(P.V[:, S])
    Y = np.linalg.solve(P.B.conj().T, np.linalg.inv(P.V).conj().T)
    V = np.asfortranarray(Y[:, S])
    assert np.linalg.norm(V.conj().T @ P.B @ U - np.eye(6)) < 1e-12
    mu = oracle.bhat_eigs(P.A, P.B, U, V, z, w)
    ref = np.sort_complex(_rho_closed(P, P.lam[S]) ** 2)
    assert np.max(np.abs(np.sort_complex(mu) - ref)) <= 1e-11


def test_count_three_inside():
    """SPEC-style example: 3 eigenvalues deep inside the unit circle, 9 far outside
    (|x| >= 4: |rho| <= 4^-16), full space: the estimate is 3; none inside: 0."""
    lam_in = np.array([0.1, -0.2 + 0.3j, 0.05j])
    lam_out = np.array([4.0, -5.0, 6j, -4.5j, 4 + 4j, -7 + 1j, 9.0, 5 - 5j, -4.2 - 3j])
    for lam, want in ((np.concatenate([lam_in, lam_out]), 3), (lam_out, 0)):
        n = len(lam)
        rng = np.random.default_rng(3)
        Vm = np.eye(n) + 0.1 * (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(n)
        A = np.asfortranarray(Vm @ np.diag(lam) @ np.linalg.inv(Vm))
        z, w = oracle.nodes(0.0, 1.0, 1.0, 16, 0)
        U = np.asfortranarray(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
        V = U @ np.linalg.inv(U.conj().T @ U).conj().T
        cnt, mu = oracle.count_estimate_bi(A, None, U, V, z, w)
        assert cnt == want, (cnt, np.abs(mu[:5]))


def test_bifeast_monitors_and_count_at_convergence():
    n, m0 = 160, 24
    P = synth.make_pencil("C4", n=n, m0=m0)
    s = P.spec
    z, w = oracle.nodes(s.c, s.r, s.aspect, s.n_e, s.rule)
    X = P.X0
    V = _bi_start(P, X)
    for _ in range(4):
        Xp, Vp = X, V
        out = oracle.feast_iterate(P.A, P.B, X, V, z, w, s.c, s.r, s.aspect)
        X, V = out["X"], out["V"]
    inside = P.lam[np.abs(P.lam - s.c) < s.r]
    res, tr, nc = oracle.monitors(out)
    assert nc == len(inside) >= 1
    assert abs(tr - inside.sum()) <= 1e-10 * s.r * nc
    assert 0 <= res <= 1e-9
    # count estimate from the last iteration's steps 4-5 (inputs V^(k-1), U^(k-1), V^H B U = I)
    assert np.linalg.norm(Vp.conj().T @ Xp - np.eye(m0)) < 1e-8
    cnt, mu = oracle.count_estimate_bi(P.A, None, Xp, Vp, z, w)
    assert cnt == len(inside)
    # the leading eigenvalues are rho(lambda)^2 of the inside eigenvalues (converged subspace)
    lead = np.sort_complex(mu[:len(inside)])
    ref = np.sort_complex(_rho_closed(P, inside) ** 2)
    assert np.max(np.abs(lead - ref)) <= 1e-8


def test_filter_gap_closed_form_ordering():
    """Unit circle, midpoint rule q = 8: |rho(r e^{i th})| = 1 / |1 + r^8 e^{8 i th}|.  On the
    real axis (th = 0) |rho| = 1/(1 + r^8) decreases with r: radii 0.1 .. 3 keep their order,
    m = 3 (r < 1), m' = 3, eps = |gamma_5 / gamma_3| for p = 4."""
    z, w = oracle.nodes(0.0, 1.0, 1.0, 8, 0)
    r = np.array([0.9, 0.1, 3.0, 1.1, 0.5, 1.5])
    lam = r.astype(complex)
    rep = oracle.filter_gap(z, w, lam, 4, np.abs(lam) < 1)
    g = 1.0 / (1.0 + r ** 8)
    assert list(rep["order"]) == [1, 4, 0, 3, 5, 2]
    assert np.allclose(rep["abs_sorted"], np.sort(g)[::-1], rtol=1e-12, atol=0)
    assert rep["m"] == 3 and rep["m_prime"] == 3
    assert abs(rep["eps"] - (1 / (1 + 1.5 ** 8)) / (1 / (1 + 0.9 ** 8))) < 1e-13
    assert abs(rep["log10_gap"] - np.log10((1 / (1 + 1.5 ** 8)) / (1 / (1 + 0.9 ** 8)))) < 1e-12


def test_filter_gap_outside_dominant_and_empty():
    """An OUTSIDE eigenvalue at r = 1.05 on the ray th = pi/8 (x^8 = -1.05^8): |rho| =
    1/(1.05^8 - 1) = 2.09 ranks first; an inside one at r = 0.95 on th = 0 has |rho| =
    1/(1 + 0.95^8) = 0.601, below the outside r = 1.2, th = pi/8 one (1/(1.2^8 - 1) = 0.435)? no:
    0.601 > 0.435 — so the sorted order is [out 1.05, in 0.1, in 0.95, out 1.2], m = 2, m' = 3;
    all eigenvalues outside: m = m' = 0."""
    z, w = oracle.nodes(0.0, 1.0, 1.0, 8, 0)
    e = np.exp(1j * np.pi / 8)
    lam = np.array([0.95, 1.2 * e, 0.1, 1.05 * e])
    rep = oracle.filter_gap(z, w, lam, 3, np.abs(lam) < 1)
    assert list(rep["order"]) == [3, 2, 0, 1]
    ref = np.array([1 / (1.05 ** 8 - 1), 1 / (1 + 0.1 ** 8), 1 / (1 + 0.95 ** 8), 1 / (1.2 ** 8 - 1)])
    assert np.allclose(rep["abs_sorted"], ref, rtol=1e-12, atol=0)
    assert rep["m"] == 2 and rep["m_prime"] == 3
    assert abs(rep["eps"] - ref[3] / ref[2]) < 1e-12
    rep = oracle.filter_gap(z, w, np.array([2.0, 3j, -4.0]), 1, np.zeros(3, bool))
    assert rep["m"] == 0 and rep["m_prime"] == 0 and np.isnan(rep["eps"])


def test_filter_gap_ties_extend_m_prime():
    """Equal |gamma| across the last inside position: m' extends to the end of the tie (a strict
    gap |gamma_{m'+1}| < |gamma_{m'}| is required; a relative difference <= 1e-12 is a
    tie, reading R22).  Conjugate points on the real-axis-symmetric circle filter have equal |rho|
    (up to rounding)."""
    z, w = oracle.nodes(0.0, 1.0, 1.0, 8, 0)
    lam = np.array([0.3 + 0.6j, 0.8 + 0.8j, 0.8 - 0.8j, 2.0])   # 0.8 +- 0.8i: |x| = 1.13 > 1, outside
    inside = np.abs(lam) < 1
    rep = oracle.filter_gap(z, w, lam, 3, inside)
    a = rep["abs_sorted"]
    assert abs(a[1] - a[2]) <= 1e-14 * a[1]
    assert rep["m"] == 1
    # inside point first, then the conjugate pair tied
    assert rep["order"][0] == 0 and rep["m_prime"] == 1
    lam2 = np.array([0.8 + 0.8j, 0.8 - 0.8j, 0.5j, 2.0])        # make the tie straddle an inside one
    rep2 = oracle.filter_gap(z, w, lam2, 3, np.array([True, False, True, False]))
    assert rep2["m"] == 2 and rep2["m_prime"] >= 3
