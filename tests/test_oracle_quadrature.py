"""Pins of oracle step O1 (quadrature rules, poles/weights, the rational filter rho).

Pinned against closed forms that do not reuse the oracle's formulas:
  * Gauss–Legendre K = 1, 2, 3 closed forms and exactness on monomials
    t^d, d <= 2K-1, vs the exact integral 2/(d+1) (even d), 0 (odd d).
  * endpoint trapezoid K = 2, 3, K = 5 integral of t^2 = 0.75.
  * midpoint trapezoid on a circle: rho = 1/(1 + x^q), x = (mu - c)/R (reading R1).
  * endpoint trapezoid on a circle: rho = 1/(1 - x^q), q = 2(K-1).
  * S:181-192 worked example: K = 3 endpoint rule on the unit circle -> poles {+-1, +-i},
    rho(0) = 1, rho(2) = -1/15, rho(0.5) = 1.0666667, rho(3) = -0.0125 (golden file).
  * shift/scale covariance rho(mu) = rho_ref((mu - c)/R).
  * Cauchy limit: rho -> 1 inside, 0 outside as K grows (eq. cauchy_contour).
  * GL K = 8 circle eta(0.5) > 0.99, eta(2) < 1e-2 (eta of P:394-401).
"""
import json
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_gl_closed_forms():
    t, w = oracle.gauss_legendre(1)
    assert np.allclose(t, [0.0], atol=1e-15) and np.allclose(w, [2.0], atol=1e-15)
    t, w = oracle.gauss_legendre(2)
    assert np.allclose(t, [-1 / np.sqrt(3), 1 / np.sqrt(3)], atol=1e-15)
    assert np.allclose(w, [1.0, 1.0], atol=1e-15)
    t, w = oracle.gauss_legendre(3)
    assert np.allclose(t, [-np.sqrt(0.6), 0.0, np.sqrt(0.6)], atol=1e-15)
    assert np.allclose(w, [5 / 9, 8 / 9, 5 / 9], atol=1e-15)


@pytest.mark.parametrize("K", [1, 2, 4, 8, 12, 16, 24, 32])
def test_gl_exact_on_monomials(K):
    t, w = oracle.gauss_legendre(K)
    assert np.all(np.diff(t) > 0) and np.all(w > 0)
    for d in range(2 * K):
        exact = 0.0 if d % 2 else 2.0 / (d + 1)
        assert abs(np.sum(w * t ** d) - exact) < 1e-13, (K, d)


def test_trapezoid_endpoint_examples():
    t, w = oracle.trapezoid_endpoint(2)
    assert np.allclose(t, [-1, 1]) and np.allclose(w, [1, 1])
    t, w = oracle.trapezoid_endpoint(3)
    assert np.allclose(t, [-1, 0, 1]) and np.allclose(w, [0.5, 1, 0.5])
    t, w = oracle.trapezoid_endpoint(5)
    assert abs(w.sum() - 2) < 1e-15 and abs(np.sum(w * t ** 2) - 0.75) < 1e-15


def _mu_samples(c, R, seed=0, k=200):
    rng = np.random.default_rng(seed)
    r = rng.uniform(0, 2.5, k)
    r = r[np.abs(r - 1) > 0.05]
    th = rng.uniform(0, 2 * np.pi, len(r))
    return c + R * r * np.exp(1j * th)


@pytest.mark.parametrize("q,c,R", [(8, 0.0, 0.5), (16, 0.2 + 0.1j, 0.3), (32, 0.5, 0.25), (16, 0.0, 0.2), (4, 0, 1)])
def test_midpoint_circle_closed_form(q, c, R):
    z, w = oracle.nodes(c, R, 1.0, q, 0)
    assert len(z) == q
    mu = _mu_samples(c, R)
    x = (mu - c) / R
    ref = 1.0 / (1.0 + x ** q)
    assert np.max(np.abs(oracle.rho(z, w, mu) - ref)) < 1e-13
    # poles at theta_j = 2 pi (j + 1/2)/q, weights (z_j - c)/q
    th = np.sort(np.mod(np.angle(z - c), 2 * np.pi))
    assert np.allclose(th, 2 * np.pi * (np.arange(q) + 0.5) / q, atol=1e-14)
    assert np.allclose(w, (z - c) / q, atol=1e-16)


@pytest.mark.parametrize("K", [3, 5, 9, 17])
def test_endpoint_circle_closed_form(K):
    q = 2 * (K - 1)
    z, w = oracle.nodes(0.0, 1.0, 1.0, q, 1)
    assert len(z) == q                       # q = 2(K-1) when +-1 are nodes
    mu = _mu_samples(0.0, 1.0, seed=K)
    ref = 1.0 / (1.0 - mu ** q)
    assert np.max(np.abs(oracle.rho(z, w, mu) - ref)) < 1e-12
    assert abs(oracle.rho(z, w, [0.0])[0] - 1.0) < 1e-14


def test_spec_worked_example_golden():
    g = json.load(open(os.path.join(GOLD, "filter_trapezoid_k3_unit_circle.json")))
    z, w = oracle.nodes(0.0, 1.0, 1.0, 4, 1)
    want = np.array([complex(*p) for p in g["poles"]])
    for p in want:
        assert np.min(np.abs(z - p)) < 1e-15
    for mu, val in g["rho"]:
        got = oracle.rho(z, w, [complex(*mu)])[0]
        assert abs(got - val) < 1e-7, (mu, got, val)


@pytest.mark.parametrize("rule,n_e", [(2, 8), (0, 16), (1, 16)])
@pytest.mark.parametrize("a", [1.0, 0.5, 0.15])
def test_shift_scale_covariance(rule, n_e, a):
    c, R = 0.3 - 0.2j, 0.7
    z, w = oracle.nodes(c, R, a, n_e, rule)
    z0, w0 = oracle.nodes(0.0, 1.0, a, n_e, rule)
    mu = _mu_samples(c, R, seed=3)
    assert np.max(np.abs(oracle.rho(z, w, mu) - oracle.rho(z0, w0, (mu - c) / R))) < 1e-12


def test_cauchy_limit_and_counts():
    inside = np.array([0.0, 0.3 + 0.2j, -0.5j])
    outside = np.array([1.6, -2.0 + 1j, 3j])
    prev_in = prev_out = None
    for K in (4, 8, 16, 32):
        z, w = oracle.nodes(0.0, 1.0, 1.0, K, 2)
        assert len(z) == 2 * K               # q = 2K for Gauss–Legendre
        ei = np.max(np.abs(oracle.rho(z, w, inside) - 1))
        eo = np.max(np.abs(oracle.rho(z, w, outside)))
        if prev_in is not None:
            assert ei < prev_in and eo < prev_out
        prev_in, prev_out = ei, eo
    assert prev_in < 1e-6 and prev_out < 1e-6


def test_gl8_eta_spec():
    z, w = oracle.nodes(0.0, 1.0, 1.0, 8, 2)
    th = np.linspace(0, 2 * np.pi, 1024, endpoint=False)
    eta_in = np.min(np.abs(oracle.rho(z, w, 0.5 * np.exp(1j * th))))
    eta_out = np.max(np.abs(oracle.rho(z, w, 2.0 * np.exp(1j * th))))
    assert eta_in > 0.99 and eta_out < 1e-2


def test_ellipse_semi_axes():
    # reading R2: semi-axes R (real) and R*a (imaginary), C3's ellipse
    z, w = oracle.nodes(0.0, 0.4, 0.15, 16, 2)
    assert len(z) == 32
    assert np.max(np.abs(z.real)) < 0.4 and np.max(np.abs(z.real)) > 0.399
    assert np.max(np.abs(z.imag)) < 0.06 and np.max(np.abs(z.imag)) > 0.059
    assert np.allclose((z.real / 0.4) ** 2 + (z.imag / 0.06) ** 2, 1.0, atol=1e-14)


def test_bad_arguments():
    with pytest.raises(ValueError):
        oracle.nodes(0, -1, 1, 8, 0)
    with pytest.raises(ValueError):
        oracle.nodes(0, 1, 1, 7, 0)   # midpoint needs an even pole count (two halves)


# ---------------------------------------------------------------- composite contours (NEXT-4)
SQUARE = [("line", 1 - 1j, 1 + 1j), ("line", 1 + 1j, -1 + 1j), ("line", -1 + 1j, -1 - 1j), ("line", -1 - 1j, 1 - 1j)]
TRIANGLE = [("line", -1, 1), ("line", 1, 1j), ("line", 1j, -1)]
SEMICIRCLE = [("arc", 0, 1.0, 0.0, np.pi), ("line", -1, 1)]


@pytest.mark.parametrize("segs", [SQUARE, TRIANGLE])
def test_composite_polygon_moments_vanish(segs):
    """Closed polygon, Gauss-Legendre K per side: sum_j w_j z_j^k = (1/2 pi i) oint z^k dz = 0
    exactly for k <= 2K - 2 (phi linear on each side, so z^k phi' has degree k <= 2K - 1 in t)."""
    K = 5
    z, w = oracle.contour_nodes(segs, K, 2)
    for k in range(2 * K - 1):
        assert abs(np.sum(w * z ** k)) <= 1e-13 * max(1.0, np.max(np.abs(z)) ** k)


def test_composite_full_circle_arc_equals_midpoint_rule():
    """One arc of angle 2 pi with the midpoint rule reproduces the midpoint trapezoid on the circle
    (reading R1): the same poles and weights from two different constructions."""
    c, R, q = 0.3 - 0.2j, 0.7, 12
    z1, w1 = oracle.contour_nodes([("arc", c, R, 0.0, 2 * np.pi)], q, 0)
    z2, w2 = oracle.nodes(c, R, 1.0, q, 0)
    o1, o2 = np.argsort(np.angle(z1 - c)), np.argsort(np.angle(z2 - c))
    assert np.max(np.abs(z1[o1] - z2[o2])) < 1e-14 and np.max(np.abs(w1[o1] - w2[o2])) < 1e-15


def test_composite_spec_examples():
    """S:210-218 examples: square inside(0); triangle (-1, 1, i) with the trapezoid (midpoint, R18)
    K = 8 per segment: |rho(centroid) - 1| <= 0.05; semicircle (arc + diameter): rho ~ 1 at 0.5i,
    ~ 0 at -0.5i; and the Cauchy limit rho -> 1 inside / 0 outside as K grows."""
    z, w = oracle.contour_nodes(SQUARE, 8, 2)
    assert abs(oracle.rho(z, w, [0.0])[0] - 1) < 1e-5 and abs(oracle.rho(z, w, [3.0])[0]) < 1e-9
    z, w = oracle.contour_nodes(TRIANGLE, 8, 0)
    assert abs(oracle.rho(z, w, [1j / 3])[0] - 1) <= 0.05
    z, w = oracle.contour_nodes(SEMICIRCLE, 16, 2)
    r_in, r_out = oracle.rho(z, w, [0.5j, -0.5j])
    assert abs(r_in - 1) < 1e-6 and abs(r_out) < 1e-6
    errs = [abs(oracle.rho(*oracle.contour_nodes(TRIANGLE, K, 0), [1j / 3])[0] - 1) for K in (4, 8, 16, 32)]
    assert all(b < a for a, b in zip(errs, errs[1:]))


# ---------------------------------------------------------------- ellipse weights, aspect != 1
# eq. ellipses and eq. quadrature_for_pi: sigma = w_k phi'(t)/(2 pi i) with
# phi'(t) = (pi/2) R (-sin th + i a cos th).  These pins bind the aspect a inside the derivative
# (dropping it leaves the pole positions, and every a = 1 pin, unchanged).
ELLIPSES = [(0.3 - 0.1j, 0.4, 0.15), (0.0, 0.4, 0.15), (0.5 + 0.2j, 1.3, 0.5), (-0.2j, 0.25, 2.0)]


@pytest.mark.parametrize("c,R,a", ELLIPSES)
@pytest.mark.parametrize("rule,n_e", [(0, 8), (0, 16), (0, 32), (1, 16)])
def test_ellipse_moments_vanish_exactly(c, R, a, rule, n_e):
    """The midpoint and endpoint trapezoid rules are the q-point periodic trapezoid rule in
    theta, exact on trigonometric polynomials of degree <= q - 1.  (z - c)^k phi'(theta) has
    degree k + 1, so sum_j w_j (z_j - c)^k = (1/2 pi i) oint (z - c)^k dz = 0 for k <= q - 2
    (Cauchy's theorem), for every aspect a."""
    z, w = oracle.nodes(c, R, a, n_e, rule)
    q = len(z)
    assert q == n_e
    for k in range(q - 1):
        scale = np.sum(np.abs(w) * np.abs(z - c) ** k)
        assert abs(np.sum(w * (z - c) ** k)) <= 1e-14 * scale, (k, a)


@pytest.mark.parametrize("c,R,a", ELLIPSES + [(0.1, 0.7, 1.0)])
@pytest.mark.parametrize("rule,n_e", [(0, 8), (0, 16), (1, 16), (2, 8), (2, 16)])
def test_ellipse_area_identity(c, R, a, rule, n_e):
    """Green's theorem: oint conj(z - c) dz = 2i * Area, so (1/2 pi i) oint conj(z - c) dz =
    Area / pi = R * (R a) = R^2 a for the ellipse with semi-axes R and R a (reading R2).  The
    trapezoid rules integrate this degree-2 trigonometric polynomial exactly; Gauss-Legendre on
    the two halves integrates the entire function of t to rounding at K >= 8."""
    z, w = oracle.nodes(c, R, a, n_e, rule)
    assert abs(np.sum(w * np.conj(z - c)) - R * R * a) <= 1e-14 * R * R


@pytest.mark.parametrize("rule", [0, 2])
@pytest.mark.parametrize("a", [0.15, 0.5])
def test_ellipse_cauchy_limit(rule, a):
    """Cauchy's integral formula (eq. cauchy_contour) on thin ellipses: rho -> 1 at
    points inside, -> 0 outside, monotonically as K grows, to 1e-8 at K = 256 per half."""
    c, R = 0.3 - 0.1j, 0.4
    inside = c + R * np.array([0.0, 0.3, 0.5j * a, -0.2 + 0.1j * a])
    outside = c + R * np.array([1.6, 3j * a, -2.0, 1.2 + 0.5j])
    prev = None
    for K in (8, 16, 32, 64, 128, 256):
        z, w = oracle.nodes(c, R, a, 2 * K if rule == 0 else K, rule)
        err = max(np.max(np.abs(oracle.rho(z, w, inside) - 1)), np.max(np.abs(oracle.rho(z, w, outside))))
        if prev is not None and prev > 1e-13:
            assert err < prev, (K, err, prev)
        prev = err
    assert prev < 1e-8
