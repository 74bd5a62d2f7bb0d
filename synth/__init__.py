"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic (no quadrature, no filter, no shifted
solve, no Rayleigh–Ritz): it only draws the pencils (A, B), the starting blocks X0 and the
known eigen-data (lambda, V) of BASELINE.json configs C1..C5, following the recipe in
DESIGN.md §"Input recipe".  Seeds: seed_k = 14042891 + k for config k;
numpy SeedSequence(seed_k).spawn(4) -> streams [lambda, G(V), G_B or (G_H, D, G_S), X0],
each Generator(PCG64).  Complex Gaussians are CN(0,1) = (N(0,1) + i N(0,1)) / sqrt(2).

Dense matrices are numpy complex128 in Fortran (column-major) order.  Building A needs
V^{-1}; that is a library solve (numpy LAPACK, or torch.linalg on a GPU for n >= 8192),
not part of the method.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

SEED_BASE = 14042891

# rule ids (same numbering as include/feast.h and the oracle)
RULE_TRAPEZOID = 0          # midpoint-offset trapezoid on the circle (reading R1)
RULE_TRAPEZOID_ENDPOINT = 1  # paper's K-point rule with both endpoints
RULE_GAUSS_LEGENDRE = 2      # K nodes per half, q = 2K


@dataclasses.dataclass(frozen=True)
class ConfigSpec:
    key: str
    n: int
    m0: int
    kind: str            # "std", "gen", "csym", "bi", "gen"
    c: complex
    r: float             # real semi-axis R
    aspect: float        # a: imaginary semi-axis = R * a (reading R2)
    n_e: int
    rule: int
    mode: str            # "right" | "bi"
    iters: int
    vscale: float        # V = I + vscale * G / sqrt(n)
    bscale: float        # B = I + bscale * G_B / sqrt(n) (0 => B = I)
    lam: str             # eigenvalue distribution

    @property
    def q(self) -> int:
        return 2 * self.n_e if self.rule == RULE_GAUSS_LEGENDRE else self.n_e

    @property
    def b_is_identity(self) -> bool:
        return self.kind in ("std", "bi")

    @property
    def real_pencil(self) -> bool:
        return self.kind == "gen_real"


# BASELINE.json configs[0..4] (C1..C5)
CONFIGS = {
    "C1": ConfigSpec("C1", 200, 64, "std", 0j, 0.5, 1.0, 8, RULE_TRAPEZOID, "right", 10, 0.1, 0.0, "square1"),
    "C2": ConfigSpec("C2", 2048, 128, "gen", 0.2 + 0.1j, 0.3, 1.0, 16, RULE_TRAPEZOID, "right", 8, 0.1, 0.01, "disk1"),
    "C3": ConfigSpec("C3", 8192, 256, "csym", 0j, 0.4, 0.15, 16, RULE_GAUSS_LEGENDRE, "right", 6, 0.0, 0.01, "none"),
    "C4": ConfigSpec("C4", 16384, 512, "bi", 0.5 + 0j, 0.25, 1.0, 32, RULE_TRAPEZOID, "bi", 5, 0.05, 0.0, "rect2x1"),
    "C5": ConfigSpec("C5", 32768, 1024, "gen", 0j, 0.2, 1.0, 16, RULE_TRAPEZOID, "right", 4, 0.05, 0.005, "disk1"),
    # Companion (NOT a BASELINE config): a REAL generalized pencil of C2's size, standing in for the
    # paper's real non-symmetric application pencils; contour centred on the real axis so the
    # poles come in conjugate pairs (real-pencil mode, SURVEY NEXT-2b).  B = I + 0.01 G_B/sqrt(n),
    # V = I + 0.1 G/sqrt(n) with REAL Gaussians; eigenvalues in conjugate pairs a +- ib, (a, b)
    # uniform in the upper half of the unit disk; A = B V Lr V^-1 with Lr = blockdiag([[a, b], [-b, a]]).
    "R2": ConfigSpec("R2", 2048, 128, "gen_real", 0.2 + 0j, 0.3, 1.0, 16, RULE_TRAPEZOID, "right", 8, 0.1, 0.01,
                     "pairs_disk1"),
}


def _cn(rng: np.random.Generator, shape) -> np.ndarray:
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) / math.sqrt(2.0)


@dataclasses.dataclass
class Pencil:
    spec: ConfigSpec
    n: int
    m0: int
    A: np.ndarray
    B: np.ndarray | None      # None means identity
    X0: np.ndarray
    lam: np.ndarray | None    # known eigenvalues (None for C3)
    V: np.ndarray | None      # known right eigenvectors of B^-1 A (None for C3)

    @property
    def q(self) -> int:
        return self.spec.q


def make_pencil(key: str, n: int | None = None, m0: int | None = None, seed_offset: int = 0) -> Pencil:
    """Draw config `key` (C1..C5) at its BASELINE size, or a same-recipe shadow of size n
    (and block width m0).  Deterministic in (key, n, m0, seed_offset)."""
    spec = CONFIGS[key]
    n = spec.n if n is None else int(n)
    m0 = spec.m0 if m0 is None else int(m0)
    k = int(key[1:]) - 1 + (100 if key.startswith("R") else 0)
    ss = np.random.SeedSequence(SEED_BASE + k + 1000 * seed_offset)
    r_lam, r_v, r_b, r_x = (np.random.Generator(np.random.PCG64(s)) for s in ss.spawn(4))
    sq = math.sqrt(n)
    lam = V = None
    if spec.kind == "gen_real":
        if n % 2:
            raise ValueError("gen_real needs an even n (conjugate eigenvalue pairs)")
        h = n // 2
        rr = np.sqrt(r_lam.uniform(0, 1, h))
        th = math.pi * r_lam.uniform(0, 1, h)
        a, b = rr * np.cos(th), rr * np.sin(th)
        Vr = np.eye(n) + spec.vscale * r_v.standard_normal((n, n)) / sq
        Lr = np.zeros((n, n))
        idx = np.arange(h)
        Lr[2 * idx, 2 * idx] = a
        Lr[2 * idx + 1, 2 * idx + 1] = a
        Lr[2 * idx, 2 * idx + 1] = b
        Lr[2 * idx + 1, 2 * idx] = -b
        M = np.linalg.solve(Vr.T, (Vr @ Lr).T).T          # V Lr V^-1 (library solve)
        Br = np.eye(n) + spec.bscale * r_b.standard_normal((n, n)) / sq
        A = np.asfortranarray((Br @ M).astype(np.complex128))
        B = np.asfortranarray(Br.astype(np.complex128))
        lam = np.empty(n, dtype=np.complex128)
        lam[0::2] = a + 1j * b
        lam[1::2] = a - 1j * b
        V = np.empty((n, n), dtype=np.complex128)           # eigenvectors of B^-1 A: V [1, +-i]
        V[:, 0::2] = Vr[:, 0::2] + 1j * Vr[:, 1::2]
        V[:, 1::2] = Vr[:, 0::2] - 1j * Vr[:, 1::2]
        V = np.asfortranarray(V)
        X0 = np.asfortranarray(_cn(r_x, (n, m0)))
        return Pencil(spec, n, m0, A, B, X0, lam, V)
    if spec.kind == "csym":
        gh = r_b.standard_normal((n, n))
        H = (gh + gh.T) / (2.0 * sq)
        D = r_b.uniform(0.0, 0.05, n)
        gs = r_b.standard_normal((n, n))
        S = (gs + gs.T) / (2.0 * sq)
        A = np.asfortranarray(H + 1j * np.diag(D))
        B = np.asfortranarray((np.eye(n) + spec.bscale * S).astype(np.complex128))
    else:
        if spec.lam == "square1":
            lam = r_lam.uniform(-1, 1, n) + 1j * r_lam.uniform(-1, 1, n)
        elif spec.lam == "rect2x1":
            lam = r_lam.uniform(-2, 2, n) + 1j * r_lam.uniform(-1, 1, n)
        elif spec.lam == "disk1":
            rr = np.sqrt(r_lam.uniform(0, 1, n))
            th = 2 * math.pi * r_lam.uniform(0, 1, n)
            lam = rr * np.exp(1j * th)
        else:
            raise ValueError(spec.lam)
        V = np.eye(n, dtype=np.complex128) + spec.vscale * _cn(r_v, (n, n)) / sq
        # A = B V diag(lam) V^-1 :  (V diag(lam)) V^-1 = solve(V^T, (V diag(lam))^T)^T
        M = np.linalg.solve(V.T, (V * lam[None, :]).T).T
        if spec.b_is_identity:
            B = None
            A = np.asfortranarray(M)
        else:
            B = np.asfortranarray(np.eye(n) + spec.bscale * _cn(r_b, (n, n)) / sq)
            A = np.asfortranarray(B @ M)
        V = np.asfortranarray(V)
    X0 = np.asfortranarray(_cn(r_x, (n, m0)))
    return Pencil(spec, n, m0, A, B, X0, lam, V)


def node_owner_range(q: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous node block owned by `rank` (reading R17): [r q/P, (r+1) q/P)."""
    if world < 1 or q % world:
        raise ValueError(f"q={q} not divisible by world={world}")
    per = q // world
    return rank * per, (rank + 1) * per


def random_block(n: int, m: int, seed: int) -> np.ndarray:
    return np.asfortranarray(_cn(np.random.Generator(np.random.PCG64(seed)), (n, m)))


def make_pencil_torch(key: str, n: int | None = None, m0: int | None = None, device="cuda", seed_offset: int = 0):
    """GPU variant of make_pencil for the large configs (C3-C5 at full size): the same recipe
    drawn with torch's seeded generator on the device, and A built with a library solve
    (torch.linalg.solve, cuSOLVER) — fixture generation, not the method.  Returns a Pencil
    whose matrices are column-major complex128 torch tensors on `device` (V and lam kept for
    the spectral identity, on the device as well)."""
    import torch

    spec = CONFIGS[key]
    n = spec.n if n is None else int(n)
    m0 = spec.m0 if m0 is None else int(m0)
    k = int(key[1:]) - 1
    g = torch.Generator(device=device)
    g.manual_seed(SEED_BASE + k + 1000 * seed_offset + 7)
    sq = math.sqrt(n)
    f64 = dict(dtype=torch.float64, device=device)

    def cn(shape):
        return torch.complex(torch.randn(shape, generator=g, **f64), torch.randn(shape, generator=g, **f64)) / math.sqrt(2.0)

    def colmajor(t):
        return t.t().contiguous().t()

    lam = V = None
    if spec.kind == "csym":
        gh = torch.randn((n, n), generator=g, **f64)
        H = (gh + gh.T) / (2.0 * sq)
        del gh
        D = torch.rand(n, generator=g, **f64) * 0.05
        A = torch.complex(H, torch.diag(D))
        del H
        gs = torch.randn((n, n), generator=g, **f64)
        B = torch.eye(n, **f64) + spec.bscale * (gs + gs.T) / (2.0 * sq)
        del gs
        B = torch.complex(B, torch.zeros_like(B))
        A, B = colmajor(A), colmajor(B)
    else:
        if spec.lam == "square1":
            lam = torch.complex(torch.rand(n, generator=g, **f64) * 2 - 1, torch.rand(n, generator=g, **f64) * 2 - 1)
        elif spec.lam == "rect2x1":
            lam = torch.complex(torch.rand(n, generator=g, **f64) * 4 - 2, torch.rand(n, generator=g, **f64) * 2 - 1)
        else:
            rr = torch.sqrt(torch.rand(n, generator=g, **f64))
            th = 2 * math.pi * torch.rand(n, generator=g, **f64)
            lam = torch.polar(rr, th)
        V = cn((n, n)) * (spec.vscale / sq)
        V.diagonal().add_(1.0)
        # A = V diag(lam) V^-1 (= solve(V^T, (V diag(lam))^T)^T)
        M = torch.linalg.solve(V.T, (V * lam[None, :]).T).T
        if spec.b_is_identity:
            B = None
            A = colmajor(M)
        else:
            B = cn((n, n)) * (spec.bscale / sq)
            B.diagonal().add_(1.0)
            A = colmajor(B @ M)
            B = colmajor(B)
        del M
    X0 = colmajor(cn((n, m0)))
    return Pencil(spec, n, m0, A, B, X0, lam, V)
