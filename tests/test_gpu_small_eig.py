"""The one-CTA reduced eigensolver (feast_small_eig; feast_iterate's reduced problem for m0 <= 160,
R-FEAST step 5 P:511-512): eigenpairs of small dense complex matrices on the GPU, checked against
their definition M w = lambda w (residual) and LAPACK's eigenvalues (numpy), on random, structured
(diagonal, triangular, real with conjugate pairs, repeated / clustered eigenvalues) matrices."""
import numpy as np
import pytest
import torch

from paper_1404_2891_b200 import feast as fb

pytestmark = pytest.mark.gpu


def _check(M, tol_res=1e-12, tol_lam=1e-10):
    Mt = torch.from_numpy(np.asfortranarray(M.astype(np.complex128))).to("cuda")
    lam, W = fb.small_eig(Mt)
    lam, W = lam.cpu().numpy(), W.cpu().numpy()
    Wn = W / np.linalg.norm(W, axis=0, keepdims=True)
    res = np.linalg.norm(M @ Wn - Wn * lam[None, :]) / max(np.linalg.norm(M), 1e-300)
    assert res <= tol_res, res
    ref = np.linalg.eigvals(M)
    # one-to-one nearest matching (reading R14)
    used = np.zeros(len(ref), bool)
    scale = max(np.abs(ref).max(), 1e-300)
    for l in lam:
        d = np.abs(ref - l) + used * 1e300
        k = int(np.argmin(d))
        assert d[k] <= tol_lam * scale, (l, ref[k])
        used[k] = True


@pytest.mark.parametrize("m", [1, 2, 3, 17, 64, 128, 160])
def test_random_complex(m):
    rng = np.random.default_rng(m)
    _check(rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m)))


def test_structured():
    rng = np.random.default_rng(5)
    d = rng.standard_normal(40) + 1j * rng.standard_normal(40)
    _check(np.diag(d))                                               # already triangular
    _check(np.triu(rng.standard_normal((50, 50)) + 1j * rng.standard_normal((50, 50))))
    _check(rng.standard_normal((60, 60)))                            # real: conjugate pairs
    V = np.eye(48) + 0.1 * rng.standard_normal((48, 48))
    lam = np.repeat(rng.standard_normal(12) + 1j * rng.standard_normal(12), 4)   # 4-fold eigenvalues
    _check(V @ np.diag(lam) @ np.linalg.inv(V), tol_res=1e-11, tol_lam=1e-6)
    _check(np.eye(30) * (0.3 - 0.2j))                                # scalar matrix


def test_reduced_problem_shape():
    """A FEAST-like reduced matrix: B^-1 A of a pencil whose eigenvalues cluster inside a small
    disk (the filtered subspace), m0 = 128."""
    rng = np.random.default_rng(9)
    m = 128
    V = np.eye(m) + 0.1 * (rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m))) / np.sqrt(m)
    lam = 0.2 + 0.1j + 0.3 * np.sqrt(rng.uniform(0, 1, m)) * np.exp(2j * np.pi * rng.uniform(0, 1, m))
    _check(V @ np.diag(lam) @ np.linalg.inv(V))
