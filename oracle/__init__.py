"""ctypes wrapper around the plain-C oracle (oracle/feast_oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package.  It shares no code with
the product path (paper_1404_2891_b200/), and the product path never imports it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "feast_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-O2", "-fno-fast-math", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P, I64, I32, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        _lib.orc_gauss_legendre.argtypes = [I32, P, P]
        _lib.orc_trapezoid_endpoint.argtypes = [I32, P, P]
        _lib.orc_midpoint.argtypes = [I32, P, P]
        _lib.orc_nodes.argtypes = [D, D, D, D, I32, I32, P, P]
        _lib.orc_contour_nodes.argtypes = [I32, P, P, I32, I32, P, P]
        _lib.orc_rho.argtypes = [I32, P, P, I32, P, P]
        _lib.orc_rho.restype = None
        _lib.orc_lu.argtypes = [I64, P, I64, P, P]
        _lib.orc_lu_solve.argtypes = [I64, P, I64, P, I64, P, I64, I32]
        _lib.orc_lu_solve.restype = None
        _lib.orc_gemm.argtypes = [I64, I64, I64, I32, P, I64, P, I64, P, I64]
        _lib.orc_gemm.restype = None
        _lib.orc_project.argtypes = [I64, I64, P, I64, P, I64, P, I64, I32, P, P, I32, I32, I32, P, I64, P]
        _lib.orc_eig.argtypes = [I32, P, P, P, P]
        _lib.orc_threads.argtypes = [I32]
        _lib.orc_feast_iterate.argtypes = [I64, I64, P, I64, P, I64, I32, P, P, D, D, D, D,
                                           P, I64, P, I64, P, P, P, P, I32]
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _cf(a):
    return np.asfortranarray(a, dtype=np.complex128)


def gauss_legendre(K):
    t = np.zeros(K); w = np.zeros(K)
    assert lib().orc_gauss_legendre(K, _p(t), _p(w)) == 0
    return t, w


def trapezoid_endpoint(K):
    t = np.zeros(K); w = np.zeros(K)
    assert lib().orc_trapezoid_endpoint(K, _p(t), _p(w)) == 0
    return t, w


def midpoint(K):
    t = np.zeros(K); w = np.zeros(K)
    assert lib().orc_midpoint(K, _p(t), _p(w)) == 0
    return t, w


def nodes(c, R, a, n_e, rule):
    """Poles z_j and weights w_j (complex arrays of length q)."""
    z = np.zeros(2 * 4 * max(n_e, 2) + 8); w = np.zeros_like(z)
    q = lib().orc_nodes(float(np.real(c)), float(np.imag(c)), float(R), float(a), int(n_e), int(rule), _p(z), _p(w))
    if q < 0:
        raise ValueError("bad contour/rule arguments")
    return z[:2 * q].view(np.complex128).copy(), w[:2 * q].view(np.complex128).copy()


def contour_nodes(segments, K, rule):
    """Composite contour: segments = [("line", a, b) | ("arc", c, R, th0, th1)], the
    rule (0 midpoint, 2 Gauss-Legendre) with K nodes per segment.  Returns (z, w)."""
    kind = np.array([0 if s[0] == "line" else 1 for s in segments], dtype=np.int32)
    par = np.zeros(5 * len(segments))
    for i, s in enumerate(segments):
        if s[0] == "line":
            par[5 * i:5 * i + 4] = [complex(s[1]).real, complex(s[1]).imag, complex(s[2]).real, complex(s[2]).imag]
        else:
            par[5 * i:5 * i + 5] = [complex(s[1]).real, complex(s[1]).imag, s[2], s[3], s[4]]
    q = len(segments) * K
    z = np.zeros(2 * q); w = np.zeros(2 * q)
    r = lib().orc_contour_nodes(len(segments), _p(kind), _p(par), int(K), int(rule), _p(z), _p(w))
    if r < 0:
        raise ValueError("bad contour/rule arguments")
    return z.view(np.complex128).copy(), w.view(np.complex128).copy()


def rho(z, w, mu):
    mu = np.atleast_1d(np.asarray(mu, dtype=np.complex128)).copy()
    z = np.ascontiguousarray(z, dtype=np.complex128); w = np.ascontiguousarray(w, dtype=np.complex128)
    out = np.zeros_like(mu)
    lib().orc_rho(len(z), _p(z), _p(w), len(mu), _p(mu), _p(out))
    return out


def lu(M):
    LU = _cf(M).copy(order="F")
    n = LU.shape[0]
    piv = np.zeros(n, dtype=np.int32); st = np.zeros(2)
    info = lib().orc_lu(n, _p(LU), n, _p(piv), _p(st))
    return LU, piv, info, st


def lu_solve(LU, piv, Bm, trans=0):
    X = _cf(Bm).copy(order="F")
    if X.ndim == 1:
        X = X.reshape(-1, 1, order="F")
    n = LU.shape[0]
    lib().orc_lu_solve(n, _p(LU), n, _p(piv), X.shape[1], _p(X), n, int(trans))
    return X


def gemm(Am, Bm, opa=0):
    Am = _cf(Am); Bm = _cf(Bm)
    m = Am.shape[0] if opa == 0 else Am.shape[1]
    k = Am.shape[1] if opa == 0 else Am.shape[0]
    C = np.zeros((m, Bm.shape[1]), dtype=np.complex128, order="F")
    lib().orc_gemm(m, Bm.shape[1], k, opa, _p(Am), Am.shape[0], _p(Bm), Bm.shape[0], _p(C), m)
    return C


def project(A, B, X, z, w, j0=0, j1=None, left=False, stats=False):
    """sum_j w_j (z_j B - A)^-1 (B X)  (left: sum_j conj(w_j) (z_j B - A)^-H (B^H X))."""
    A = _cf(A); X = _cf(X); Bf = None if B is None else _cf(B)
    n, m0 = X.shape
    q = len(z)
    j1 = q if j1 is None else j1
    z = np.ascontiguousarray(z, dtype=np.complex128); w = np.ascontiguousarray(w, dtype=np.complex128)
    Q = np.zeros((n, m0), dtype=np.complex128, order="F")
    st = np.zeros(2 * q)
    err = lib().orc_project(n, m0, _p(A), n, _p(Bf), n, _p(X), n, q, _p(z), _p(w), j0, j1, int(left),
                            _p(Q), n, _p(st))
    if err:
        raise ZeroDivisionError(f"singular shifted matrix at node {-err - 1}")
    return (Q, st.reshape(q, 2)) if stats else Q


def eig(Ah, Bh):
    Ah = _cf(Ah); Bh = _cf(Bh)
    m = Ah.shape[0]
    lam = np.zeros(m, dtype=np.complex128); W = np.zeros((m, m), dtype=np.complex128, order="F")
    e = lib().orc_eig(m, _p(Ah), _p(Bh), _p(lam), _p(W))
    if e:
        raise RuntimeError(f"orc_eig failed ({e})")
    return lam, W


def feast_iterate(A, B, X, V, z, w, c, R, a, ortho=True):
    """One R-FEAST (V is None) or Bi-FEAST iteration; X (and V) updated in place copies."""
    A = _cf(A); Bf = None if B is None else _cf(B)
    X = _cf(X).copy(order="F"); V = None if V is None else _cf(V).copy(order="F")
    n, m0 = X.shape
    z = np.ascontiguousarray(z, dtype=np.complex128); w = np.ascontiguousarray(w, dtype=np.complex128)
    lam = np.zeros(m0, dtype=np.complex128); res = np.zeros(m0); resp = np.zeros(m0)
    flags = np.zeros(m0, dtype=np.int32)
    e = lib().orc_feast_iterate(n, m0, _p(A), n, _p(Bf), n, len(z), _p(z), _p(w),
                                float(np.real(c)), float(np.imag(c)), float(R), float(a),
                                _p(X), n, _p(V), n, _p(lam), _p(res), _p(resp), _p(flags), int(ortho))
    if e:
        raise RuntimeError(f"orc_feast_iterate failed ({e})")
    return dict(X=X, V=V, lam=lam, resid=res, resid_paper=resp, flags=flags)


def threads(n: int = 0) -> int:
    """Set (n > 0) and return the oracle's OpenMP team size (host timing legs only)."""
    return int(lib().orc_threads(int(n)))


# ---------------------------------------------------------------- NEXT-3: count
# estimate, candidate monitors and the filter-gap report — compositions of the primitives above
# (projectors, gemm, eig, rho), written out step by step.

def bhat_eigs(A, B, U, V, z, w):
    """Eigenvalues of V^H B U with U^ = rho(B^-1 A) U and V^ = the left projector of V (Bi-FEAST
    steps 4-5; the count estimate of P:1046-1050), sorted by decreasing modulus.
    Since V^ = B^-H rho(B^-1 A)^H B^H V (reading R4), V^^H B U^ = V^H B rho(B^-1 A)^2 U: with
    V^H B U = I its eigenvalues approximate gamma_i^2 = rho(lambda_i)^2 (exactly when U spans
    eigenvectors, or when U is square)."""
    Uh = project(A, B, U, z, w)
    Vh = project(A, B, V, z, w, left=True)
    BU = Uh if B is None else gemm(B, Uh)
    M = gemm(Vh, BU, opa=2)
    m = M.shape[0]
    mu, _ = eig(M, np.eye(m, dtype=np.complex128))
    return mu[np.argsort(-np.abs(mu), kind="stable")]


def count_estimate_bi(A, B, U, V, z, w, threshold=0.25):
    """Eigenvalue-count estimate: the number of eigenvalues mu of V^^H B U^ with
    |mu| >= threshold; 1/4 = (1/2)^2 counts the gamma_i with |rho(lambda_i)| >= 1/2, the filter's
    half height (reading R21).  Returns (count, mu sorted by decreasing modulus)."""
    mu = bhat_eigs(A, B, U, V, z, w)
    count = 0
    for x in mu:
        if abs(x) >= threshold:
            count += 1
    return count, mu


def monitors(out):
    """Res_(k) = max ||A u_j - l_j B u_j|| / ||u_j|| and trace_(k) = sum l_j over the candidates
    (inside the contour and that residual <= 1e-4) of one feast_iterate output.
    Res_(k) is -1 when there is no candidate."""
    res, tr, nc = -1.0, 0j, 0
    for j in range(len(out["lam"])):
        if out["flags"][j] & 2:
            nc += 1
            tr += out["lam"][j]
            if out["resid_paper"][j] > res:
                res = out["resid_paper"][j]
    return res, tr, nc


def filter_gap(z, w, lam, p, inside):
    """FilterGapReport (§4): gamma_j = rho(lambda_j) numbered so that |gamma_1| >= ... >=
    |gamma_n| (stable in the input order on ties); m = #{lambda_j inside C}; m' = the smallest
    l >= (last sorted position of an inside eigenvalue) with a strict gap |gamma_{l+1}| < |gamma_l|
    (or l = n), a relative difference <= 1e-12 counting as a tie (reading R22); eps = |gamma_{p+1} / gamma_{m'}| and log10 |rho(lambda_{p+1}) / rho(lambda_m)|
    (SPEC S:329-332).  Returns dict(abs_sorted, order, m, m_prime, eps, log10_gap);
    eps / log10_gap are nan when p >= n or m (m') = 0."""
    lam = np.asarray(lam, dtype=np.complex128)
    n = len(lam)
    g = rho(z, w, lam)
    a = [abs(x) for x in g]
    order = sorted(range(n), key=lambda j: (-a[j], j))
    asorted = [a[j] for j in order]
    m = int(sum(1 for j in range(n) if inside[j]))
    last = 0
    for pos, j in enumerate(order, start=1):
        if inside[j]:
            last = pos
    mp = last
    while mp < n and mp > 0 and not (asorted[mp] < (1.0 - 1e-12) * asorted[mp - 1]):   # a tie is no gap (R22)
        mp += 1
    eps = asorted[p] / asorted[mp - 1] if (p < n and mp >= 1) else float("nan")
    lg = float(np.log10(asorted[p] / asorted[m - 1])) if (p < n and m >= 1) else float("nan")
    return dict(abs_sorted=np.array(asorted), order=np.array(order, dtype=np.int64), m=m, m_prime=mp, eps=eps,
                log10_gap=lg)
