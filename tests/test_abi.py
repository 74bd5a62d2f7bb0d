"""C-ABI checks that need no GPU: the library loads, exports every symbol include/feast.h
declares, validates arguments (FEAST_E_ARG) and generates the same poles/weights as the
oracle (node generation is host code in the library, written independently)."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
from paper_1404_2891_b200 import feast as fb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "feast.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(feast_[a-z_]+)\s*\(", src)) - {"feast_allreduce_fn"})


def test_exports_every_declared_symbol():
    lib = fb.load_library()
    decl = _declared()
    assert set(decl) == set(fb.EXPORTS), set(decl) ^ set(fb.EXPORTS)
    for name in decl:
        assert hasattr(lib, name), name
    assert b"sm_100a" in lib.feast_version()


def _init(n=64, m0=8, c=0j, r=1.0, a=1.0, n_e=8, rule=0, mode=0, bid=1, rank=0, world=1, batch=0):
    lib = fb.load_library()
    h = ctypes.c_void_p()
    rc = lib.feast_init(ctypes.byref(h), n, m0, c.real, c.imag, r, a, n_e, rule, mode, bid, rank, world, batch, None)
    return rc, h


@pytest.mark.parametrize("kw", [dict(n=0), dict(m0=0), dict(m0=65), dict(r=0.0), dict(r=-1.0), dict(a=0.0),
                                dict(n_e=7), dict(n_e=0, rule=2), dict(rule=3), dict(mode=2), dict(world=3),
                                dict(rank=1), dict(world=0), dict(n_e=6, rule=1, world=4), dict(n=40000)])
def test_init_rejects_bad_arguments(kw):
    rc, h = _init(**kw)
    assert rc == fb.E_ARG and not h.value


def _nodes(h):
    lib = fb.load_library()
    q = ctypes.c_int32()
    lib.feast_nodes(h, ctypes.byref(q), None, None, None, None)
    z = np.zeros(2 * q.value)
    w = np.zeros(2 * q.value)
    j0, j1 = ctypes.c_int32(), ctypes.c_int32()
    lib.feast_nodes(h, None, z.ctypes.data_as(ctypes.c_void_p), w.ctypes.data_as(ctypes.c_void_p),
                    ctypes.byref(j0), ctypes.byref(j1))
    return z.view(np.complex128), w.view(np.complex128), j0.value, j1.value


@pytest.mark.parametrize("c,r,a,n_e,rule", [(0j, 0.5, 1.0, 8, 0), (0.2 + 0.1j, 0.3, 1.0, 16, 0), (0j, 0.4, 0.15, 16, 2),
                                            (0.5, 0.25, 1.0, 32, 0), (0j, 1.0, 1.0, 4, 1), (0j, 1.0, 1.0, 16, 1),
                                            (1 - 1j, 2.0, 0.5, 5, 2)])
def test_library_nodes_match_oracle(c, r, a, n_e, rule):
    rc, h = _init(c=c, r=r, a=a, n_e=n_e, rule=rule)
    assert rc == 0
    z, w, j0, j1 = _nodes(h)
    zo, wo = oracle.nodes(c, r, a, n_e, rule)
    assert len(z) == len(zo) and (j0, j1) == (0, len(z))
    for zi, wi in zip(zo, wo):
        k = np.argmin(np.abs(z - zi))
        assert abs(z[k] - zi) < 1e-14 * max(1, r) and abs(w[k] - wi) < 1e-14 * max(1, r)
    fb.load_library().feast_destroy(h)


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_node_ownership_partition(world):
    import synth
    owned = []
    for rank in range(world):
        rc, h = _init(n_e=16, rank=rank, world=world)
        assert rc == 0
        _, _, j0, j1 = _nodes(h)
        assert (j0, j1) == synth.node_owner_range(16, rank, world)
        owned += list(range(j0, j1))
        fb.load_library().feast_destroy(h)
    assert owned == list(range(16))


def test_workspace_size_scales_with_batch():
    lib = fb.load_library()
    sizes = []
    for batch in (1, 4):
        rc, h = _init(n=512, m0=32, batch=batch)
        b = ctypes.c_size_t()
        assert lib.feast_workspace_bytes(h, ctypes.byref(b)) == 0
        sizes.append(b.value)
        lib.feast_destroy(h)
    assert sizes[1] - sizes[0] >= 3 * 16 * 512 * 512


def test_library_has_no_static_tls():
    """The .so is dlopen'ed into a process that already loaded torch/CUDA: a STATIC_TLS flag
    (initial-exec TLS, e.g. from a statically linked cudart) can fail with 'cannot allocate
    memory in static TLS block'.  The build links cudart shared to avoid it."""
    import subprocess
    out = subprocess.run(["readelf", "-d", fb.LIB_PATH], capture_output=True, text=True).stdout
    assert "STATIC_TLS" not in out
    assert "libcudart.so" in out


def test_real_pencil_units_and_guards():
    """feast_set_real_pencil: conjugate-pole orbits become the factorisation units (host logic,
    no GPU); refused for a contour off the real axis and after the workspace is bound."""
    lib = fb.load_library()
    rc, h = _init(n=64, m0=8, c=0.2 + 0j, n_e=16, rule=0, world=2, rank=1)
    assert rc == 0
    assert lib.feast_set_real_pencil(h, 1) == 0
    q, j0, j1 = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    lib.feast_nodes(h, ctypes.byref(q), None, None, ctypes.byref(j0), ctypes.byref(j1))
    assert (q.value, j0.value, j1.value) == (16, 4, 8)       # 8 orbits over 2 ranks
    lib.feast_destroy(h)
    rc, h = _init(n=64, m0=8, c=0.2 + 0.1j, n_e=16, rule=0)
    assert lib.feast_set_real_pencil(h, 1) == -1             # FEAST_E_ARG: not symmetric
    lib.feast_destroy(h)
    rc, h = _init(n=64, m0=8, c=0.0 + 0j, n_e=4, rule=1)     # endpoint rule: real poles +-1
    assert lib.feast_set_real_pencil(h, 1) == 0
    lib.feast_nodes(h, ctypes.byref(q), None, None, ctypes.byref(j0), ctypes.byref(j1))
    assert (q.value, j1.value - j0.value) == (4, 3)          # {1}, {i, -i}, {-1}
    lib.feast_destroy(h)


def _contour(lib, h, segs, K, rule):
    kind = (ctypes.c_int32 * len(segs))(*[0 if s[0] == "line" else 1 for s in segs])
    par = (ctypes.c_double * (5 * len(segs)))()
    for i, s in enumerate(segs):
        vals = ([complex(s[1]).real, complex(s[1]).imag, complex(s[2]).real, complex(s[2]).imag, 0.0]
                if s[0] == "line" else [complex(s[1]).real, complex(s[1]).imag, s[2], s[3], s[4]])
        for k, v in enumerate(vals):
            par[5 * i + k] = v
    return lib.feast_set_contour(h, len(segs), kind, par, K, rule)


@pytest.mark.parametrize("rule", [0, 2])
def test_composite_contour_nodes_match_oracle(rule):
    """NEXT-4: the library's glued-contour poles/weights (host code, written independently) equal
    the oracle's; feast_filter equals the oracle's rho; open / clockwise chains are refused."""
    lib = fb.load_library()
    tri = [("line", -1, 1), ("line", 1, 1j), ("line", 1j, -1)]
    semi = [("arc", 0.1, 0.8, 0.0, np.pi), ("line", 0.1 - 0.8, 0.1 + 0.8)]
    for segs, K in ((tri, 8), (semi, 12)):
        rc, h = _init(n=64, m0=8)
        assert _contour(lib, h, segs, K, rule) == 0
        q = ctypes.c_int32()
        lib.feast_nodes(h, ctypes.byref(q), None, None, None, None)
        z = (ctypes.c_double * (2 * q.value))()
        w = (ctypes.c_double * (2 * q.value))()
        lib.feast_nodes(h, None, z, w, None, None)
        zl = np.frombuffer(z, dtype=np.complex128)
        wl = np.frombuffer(w, dtype=np.complex128)
        zo, wo = oracle.contour_nodes(segs, K, rule)
        assert np.max(np.abs(zl - zo)) < 1e-14 and np.max(np.abs(wl - wo)) < 1e-14
        mu = np.array([0.3j, 0.1 + 0.2j, 2.0, -0.5 - 0.5j], dtype=np.complex128)
        out = np.zeros_like(mu)
        assert lib.feast_filter(h, len(mu), mu.ctypes.data_as(ctypes.c_void_p), out.ctypes.data_as(ctypes.c_void_p)) == 0
        assert np.max(np.abs(out - oracle.rho(zo, wo, mu))) < 1e-13
        lib.feast_destroy(h)
    rc, h = _init(n=64, m0=8)
    assert _contour(lib, h, [("line", -1, 1), ("line", 1, 1j)], 4, rule) == -1          # open
    assert _contour(lib, h, [("line", -1, 1j), ("line", 1j, 1), ("line", 1, -1)], 4, rule) == -1   # clockwise
    lib.feast_destroy(h)


def test_filter_endpoint_trapezoid_closed_forms():
    """feast_filter on the paper's endpoint trapezoid K = 3 (q = 4) unit circle:
    rho(0) = 1, rho(2) = -1/15, and max over |mu| = 2 of |rho| = 1/15 (the eta(2) of S:207)."""
    lib = fb.load_library()
    rc, h = _init(n=64, m0=8, c=0j, r=1.0, n_e=4, rule=1)
    th = np.linspace(0, 2 * np.pi, 1024, endpoint=False)
    mu = np.concatenate([[0.0, 2.0], 2 * np.exp(1j * th)]).astype(np.complex128)
    out = np.zeros_like(mu)
    lib.feast_filter(h, len(mu), mu.ctypes.data_as(ctypes.c_void_p), out.ctypes.data_as(ctypes.c_void_p))
    assert abs(out[0] - 1) < 1e-14 and abs(out[1] + 1 / 15) < 1e-14
    assert abs(np.max(np.abs(out[2:])) - 1 / 15) < 1e-12
    lib.feast_destroy(h)


@pytest.mark.parametrize("c,r,a,n_e,rule,p", [(0j, 1.0, 1.0, 8, 0, 4), (0.2 + 0.1j, 0.3, 1.0, 16, 0, 10),
                                              (0j, 0.4, 0.15, 16, 2, 7), (0.5, 0.25, 1.0, 32, 0, 3)])
def test_filter_gap_matches_oracle(c, r, a, n_e, rule, p):
    """feast_filter_gap (host code of the library, NEXT-3) equals the oracle's report:
    same ordering, m, m' and eps / log10 gap on random spectra around the contour."""
    lib = fb.load_library()
    rc, h = _init(c=c, r=r, a=a, n_e=n_e, rule=rule)
    assert rc == 0
    z, w, _, _ = _nodes(h)
    rng = np.random.default_rng(int(100 * r) + n_e)
    rad = rng.uniform(0, 2.2, 40)
    th = rng.uniform(0, 2 * np.pi, 40)
    lam = c + r * rad * (np.cos(th) + 1j * a * np.sin(th))
    inside = rad < 1
    ref = oracle.filter_gap(z, w, lam, p, inside)
    nl = len(lam)
    lamc = np.ascontiguousarray(lam)
    ab = np.zeros(nl)
    order = np.zeros(nl, dtype=np.int32)
    m, mp, eps, lg = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_double(), ctypes.c_double()
    assert lib.feast_filter_gap(h, nl, lamc.ctypes.data_as(ctypes.c_void_p), p, ab.ctypes.data_as(ctypes.c_void_p),
                                order.ctypes.data_as(ctypes.c_void_p), ctypes.byref(m), ctypes.byref(mp),
                                ctypes.byref(eps), ctypes.byref(lg)) == 0
    lib.feast_destroy(h)
    assert list(order) == list(ref["order"])
    # |rho| far outside is a sum of O(1) terms cancelling to ~1e-12: agreement to rounding of those
    assert np.allclose(ab, ref["abs_sorted"], rtol=1e-10, atol=1e-14)
    assert (m.value, mp.value) == (ref["m"], ref["m_prime"])
    assert abs(eps.value - ref["eps"]) <= 1e-14 + 1e-8 * abs(ref["eps"])
    assert abs(lg.value - ref["log10_gap"]) <= 1e-8
