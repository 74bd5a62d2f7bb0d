"""GPU parity of NEXT-3 against the oracle and the closed forms:
  * feast_estimate_count_bi: eig(V^^H B U^) of Bi-FEAST steps 4-5 on the full
    space (eigenvalues = rho(lambda_i)^2, closed form) and vs the oracle on a shadow;
  * feast_iterate's monitors: Res_(k), trace_(k), candidates, and the tracked count
    estimate on a converging Bi-FEAST shadow (count = m, leading eigenvalues rho(lambda)^2 of the
    known inside eigenvalues, and the oracle's eig(V^^H B U^) from the same iterate)."""
import numpy as np
import pytest

import oracle
import synth
from paper_1404_2891_b200 import Feast, feast as fb
from gpu_util import dev, host

pytestmark = pytest.mark.gpu


def _rho_closed(P, lam):
    s = P.spec
    return 1.0 / (1.0 + ((lam - s.c) / s.r) ** s.q)


def _bi_start(P, U):
    G = U.conj().T @ (U if P.B is None else P.B @ U)
    return np.asfortranarray(U @ np.linalg.inv(G).conj().T)


def _match(got, ref, tol):
    ref = list(ref)
    for x in got:
        d = np.abs(np.asarray(ref) - x)
        i = int(np.argmin(d))
        assert d[i] <= tol * max(1.0, abs(x)), (x, ref[i])
        ref.pop(i)


@pytest.mark.parametrize("key", ["C2", "C4"])
def test_count_bi_full_space(key):
    n = 48
    P = synth.make_pencil(key, n=n, m0=n)
    s = P.spec
    f = Feast(n, n, s.c, s.r, s.aspect, s.n_e, s.rule, fb.BI, P.B is None)
    U = P.X0
    V = _bi_start(P, U)
    cnt, mu, Q, QL = f.estimate_count_bi(dev(P.A), dev(P.B), dev(U), dev(V))
    assert np.all(np.diff(np.abs(mu)) <= 0)
    _match(mu, _rho_closed(P, P.lam) ** 2, 1e-9)
    z, w = oracle.nodes(s.c, s.r, s.aspect, s.n_e, s.rule)
    cnt_o, mu_o = oracle.count_estimate_bi(P.A, P.B, U, V, z, w)
    assert cnt == cnt_o == int(np.sum(np.abs(_rho_closed(P, P.lam)) >= 0.5))
    _match(mu, mu_o, 1e-9)
    rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
    assert rel(host(Q), oracle.project(P.A, P.B, U, z, w)) <= 1e-10
    assert rel(host(QL), oracle.project(P.A, P.B, V, z, w, left=True)) <= 1e-10


def test_bifeast_monitors_and_tracked_count():
    n, m0 = 400, 48
    P = synth.make_pencil("C4", n=n, m0=m0)
    s = P.spec
    z, w = oracle.nodes(s.c, s.r, s.aspect, s.n_e, s.rule)
    f = Feast(n, m0, s.c, s.r, s.aspect, s.n_e, s.rule, fb.BI, True)
    f.set_count_estimate(True)
    X, V = dev(P.X0), dev(_bi_start(P, P.X0))
    A = dev(P.A)
    for _ in range(s.iters):
        Xp, Vp = host(X), host(V)
        out = f.iterate(A, None, X, V)
    mon = f.monitors()
    inside = P.lam[np.abs(P.lam - s.c) < s.r]
    flags = np.asarray(out["flags"])
    lam = np.asarray(out["lam"])
    cand = (flags & 2).astype(bool)
    assert mon["ncand"] == cand.sum() == len(inside) >= 1
    assert abs(mon["trace_k"] - lam[cand].sum()) <= 1e-13 * len(inside)
    assert abs(mon["trace_k"] - inside.sum()) <= 1e-10 * s.r * len(inside)
    assert 0 <= mon["res_k"] <= 1e-9
    assert mon["count"] == len(inside)
    _match(mon["mu"][:len(inside)], _rho_closed(P, inside) ** 2, 1e-8)
    # the oracle's eig(V^^H B U^) from the same (GPU) iterate U^(k-1), V^(k-1)
    cnt_o, mu_o = oracle.count_estimate_bi(P.A, None, Xp, Vp, z, w)
    assert cnt_o == mon["count"]
    _match(mon["mu"][:len(inside)], mu_o[:len(inside)], 1e-9)


def test_rfeast_monitors_consistent():
    P = synth.make_pencil("C1")
    s = P.spec
    f = Feast(P.n, P.m0, s.c, s.r, s.aspect, s.n_e, s.rule, fb.RIGHT, True)
    A, X = dev(P.A), dev(P.X0)
    for _ in range(s.iters):
        out = f.iterate(A, None, X)
    mon = f.monitors()
    flags = np.asarray(out["flags"])
    lam = np.asarray(out["lam"])
    cand = (flags & 2).astype(bool)
    assert mon["ncand"] == cand.sum() >= 1
    assert abs(mon["trace_k"] - lam[cand].sum()) <= 1e-13 * cand.sum()
    assert mon["count"] == -1 and mon["mu"] is None            # R-FEAST: no bi count
    An = np.linalg.norm(P.A)
    assert mon["res_k"] <= 1e-4 and mon["res_k"] >= np.max(np.asarray(out["resid"])[cand]) * An * (1 - 1e-12)
