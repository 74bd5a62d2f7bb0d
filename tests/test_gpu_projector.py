"""GPU parity of the projector hot path (eq. Rasp, eq. Lasp): the CUDA
path through the C ABI vs the plain-C oracle on the same seeded inputs.  Bar (BASELINE
north_star): relative Frobenius error <= 1e-10 in complex128."""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_1404_2891_b200 import Feast, FeastError, feast as fb
from gpu_util import dev, host, rel

pytestmark = pytest.mark.gpu
TOL = 1e-10


def _handle(P, mode=fb.RIGHT, **kw):
    s = P.spec
    return Feast(P.n, P.m0, s.c, s.r, s.aspect, s.n_e, s.rule, mode, P.B is None, **kw)


def _oracle_nodes(P):
    s = P.spec
    return oracle.nodes(s.c, s.r, s.aspect, s.n_e, s.rule)


@pytest.mark.parametrize("key,n,m0", [("C1", None, None), ("C2", 300, 40), ("C2", 129, 7), ("C1", 64, 64),
                                      ("C3", 384, 32), ("C4", 256, 48), ("C5", 200, 33)])
def test_right_projector_parity(key, n, m0):
    P = synth.make_pencil(key, n=n, m0=m0)
    f = _handle(P)
    Q = host(f.project(dev(P.A), dev(P.B), dev(P.X0)))
    z, w = _oracle_nodes(P)
    Qo = oracle.project(P.A, P.B, P.X0, z, w)
    assert rel(Q, Qo) <= TOL
    if P.V is not None:   # spectral pin as a second reference (eq. quadf_surM)
        x = (P.lam - P.spec.c) / P.spec.r
        Qs = P.V @ ((1 / (1 + x ** P.spec.q))[:, None] * np.linalg.solve(P.V, P.X0))
        assert rel(Q, Qs) <= TOL


def test_c2_full_size_parity():
    P = synth.make_pencil("C2")
    f = _handle(P)
    Q = host(f.project(dev(P.A), dev(P.B), dev(P.X0)))
    z, w = _oracle_nodes(P)
    Qo = oracle.project(P.A, P.B, P.X0, z, w)
    assert rel(Q, Qo) <= TOL


@pytest.mark.parametrize("key,n,m0", [("C4", 256, 48), ("C2", 200, 24), ("C3", 130, 16)])
def test_left_and_bi_projector_parity(key, n, m0):
    P = synth.make_pencil(key, n=n, m0=m0)
    Vin = synth.random_block(P.n, P.m0, 11)
    z, w = _oracle_nodes(P)
    f = _handle(P, mode=fb.BI)
    QL = host(f.project_left(dev(P.A), dev(P.B), dev(Vin)))
    QLo = oracle.project(P.A, P.B, Vin, z, w, left=True)
    assert rel(QL, QLo) <= TOL
    Qb, QLb = f.project_bi(dev(P.A), dev(P.B), dev(P.X0), dev(Vin))
    assert rel(host(Qb), oracle.project(P.A, P.B, P.X0, z, w)) <= TOL
    assert rel(host(QLb), QLo) <= TOL


@pytest.mark.parametrize("rule,n_e", [(fb.RULE_TRAPEZOID_ENDPOINT, 8), (fb.RULE_GAUSS_LEGENDRE, 4)])
def test_rules(rule, n_e):
    P = synth.make_pencil("C1", n=150, m0=20)
    f = Feast(P.n, P.m0, 0j, 0.5, 1.0, n_e, rule, fb.RIGHT, True)
    z, w = oracle.nodes(0j, 0.5, 1.0, n_e, rule)
    assert rel(host(f.project(dev(P.A), None, dev(P.X0))), oracle.project(P.A, None, P.X0, z, w)) <= TOL


@pytest.mark.parametrize("n,m0", [(1, 1), (2, 1), (63, 1), (64, 5), (65, 65), (130, 3)])
def test_edge_sizes(n, m0):
    P = synth.make_pencil("C2", n=n, m0=m0)
    f = _handle(P)
    z, w = _oracle_nodes(P)
    assert rel(host(f.project(dev(P.A), dev(P.B), dev(P.X0))), oracle.project(P.A, P.B, P.X0, z, w)) <= TOL


def test_zero_block_and_batching():
    P = synth.make_pencil("C2", n=160, m0=12)
    z, w = _oracle_nodes(P)
    Qo = oracle.project(P.A, P.B, P.X0, z, w)
    for batch in (1, 3, 16):   # nodes factored concurrently; ragged last batch for 3
        f = _handle(P, max_batch=batch)
        assert rel(host(f.project(dev(P.A), dev(P.B), dev(P.X0))), Qo) <= TOL
    f = _handle(P)
    Z = f.project(dev(P.A), dev(P.B), dev(np.zeros((160, 12))))
    assert torch.count_nonzero(Z).item() == 0


@pytest.mark.parametrize("world", [2, 4, 8])
def test_virtual_ranks_partition(world):
    """Rank r's partial over its nodes (reading R17), summed over r, equals the full Q
    (the node sum the NCCL all-reduce performs)."""
    P = synth.make_pencil("C2", n=200, m0=16)
    z, w = _oracle_nodes(P)
    Qo = oracle.project(P.A, P.B, P.X0, z, w)
    tot = 0
    for r in range(world):
        f = _handle(P, rank=r, world=world, partial=True)
        part = host(f.project(dev(P.A), dev(P.B), dev(P.X0)))
        j0, j1 = synth.node_owner_range(P.q, r, world)
        assert rel(part, oracle.project(P.A, P.B, P.X0, z, w, j0, j1)) <= TOL
        tot = tot + part
    assert rel(tot, Qo) <= TOL


def test_singular_node_reported():
    # pole exactly on an eigenvalue: midpoint rule on the unit circle with q = 4 has a pole at
    # exp(i pi/4); make it an eigenvalue of a diagonal A
    p = np.exp(1j * np.pi / 4)
    A = np.diag([p, 0.1, 3.0, -0.2 + 0.1j]).astype(complex)
    f = Feast(4, 2, 0j, 1.0, 1.0, 4, fb.RULE_TRAPEZOID, fb.RIGHT, True)
    zz, _, _, _ = f.nodes()
    A[0, 0] = zz[0]
    with pytest.raises(FeastError) as e:
        f.project(dev(A), None, dev(np.eye(4)[:, :2]))
    assert e.value.code == fb.E_SINGULAR
    stats, worst = f.node_stats()
    assert worst == 0 and stats[0] == 0.0


def test_reduce_parity():
    P = synth.make_pencil("C2", n=300, m0=40)
    f = _handle(P)
    Qd = f.project(dev(P.A), dev(P.B), dev(P.X0))
    Ah, Bh = f.reduce(dev(P.A), dev(P.B), Qd)
    Q = host(Qd)
    assert rel(host(Ah), oracle.gemm(Q, oracle.gemm(P.A, Q), opa=2)) <= 1e-12
    assert rel(host(Bh), oracle.gemm(Q, oracle.gemm(P.B, Q), opa=2)) <= 1e-12


@pytest.mark.parametrize("key,n,m0", [("C2", 300, 40), ("C4", 200, 24)])
def test_register_panel_variant(monkeypatch, key, n, m0):
    """The register-chunk panel kernel (used when the panel does not fit the cluster's shared
    memory, n > 4096) forced on small sizes: same parity bar."""
    monkeypatch.setenv("FEAST_PANEL", "reg")
    P = synth.make_pencil(key, n=n, m0=m0)
    z, w = _oracle_nodes(P)
    f = _handle(P, mode=fb.BI)
    Q, QL = f.project_bi(dev(P.A), dev(P.B), dev(P.X0), dev(P.X0))
    assert rel(host(Q), oracle.project(P.A, P.B, P.X0, z, w)) <= TOL
    assert rel(host(QL), oracle.project(P.A, P.B, P.X0, z, w, left=True)) <= TOL


@pytest.mark.parametrize("nbo,lookahead", [("64", "1"), ("128", "1"), ("256", "0"), ("192", "1")])
def test_blocking_variants(monkeypatch, nbo, lookahead):
    """Outer block (trailing-update K) and lookahead variants of the two-level LU: same bar,
    on a ragged size spanning several outer blocks."""
    monkeypatch.setenv("FEAST_NBO", nbo)
    monkeypatch.setenv("FEAST_LOOKAHEAD", lookahead)
    P = synth.make_pencil("C2", n=700, m0=37)
    z, w = _oracle_nodes(P)
    f = _handle(P, mode=fb.BI)
    Q, QL = f.project_bi(dev(P.A), dev(P.B), dev(P.X0), dev(P.X0))
    assert rel(host(Q), oracle.project(P.A, P.B, P.X0, z, w)) <= TOL
    assert rel(host(QL), oracle.project(P.A, P.B, P.X0, z, w, left=True)) <= TOL


def test_factor_cache_reuse():
    """NEXT-1: with the factor cache on, a second projection with the same pencil
    skips the shift + LU (fewer launches) and still matches the oracle for a new block."""
    P = synth.make_pencil("C2", n=330, m0=20)
    z, w = _oracle_nodes(P)
    f = _handle(P, mode=fb.BI)
    f.factor_cache(True)
    A, B = dev(P.A), dev(P.B)
    X1, X2 = P.X0, synth.random_block(P.n, P.m0, 99)
    Q1 = f.project(A, B, dev(X1))
    n_factor = f.last_launch_count
    Q2 = f.project(A, B, dev(X2))
    n_reuse = f.last_launch_count
    assert n_reuse < n_factor / 2
    assert rel(host(Q1), oracle.project(P.A, P.B, X1, z, w)) <= TOL
    assert rel(host(Q2), oracle.project(P.A, P.B, X2, z, w)) <= TOL
    QL = f.project_left(A, B, dev(X2))
    assert rel(host(QL), oracle.project(P.A, P.B, X2, z, w, left=True)) <= TOL
    # a different pencil (new A pointer) refactors
    A2 = dev(P.A + 0.01 * np.eye(P.n))
    Q3 = f.project(A2, B, dev(X2))
    assert f.last_launch_count >= n_factor - 2
    assert rel(host(Q3), oracle.project(P.A + 0.01 * np.eye(P.n), P.B, X2, z, w)) <= TOL


def test_graph_replay_reads_current_inputs():
    """Repeated calls with the same buffers are captured into a CUDA graph (2nd call) and replayed
    (3rd on): every call must still project the CURRENT contents of A, B and X."""
    P = synth.make_pencil("C2", n=260, m0=24)
    z, w = _oracle_nodes(P)
    f = _handle(P)
    A, B, X = dev(P.A), dev(P.B), dev(P.X0)
    Q = torch.empty_like(X)
    launches = []
    for it in range(4):
        Xh = synth.random_block(P.n, P.m0, 500 + it)
        Ah = P.A + (0.002 * it) * np.eye(P.n)
        X.copy_(dev(Xh))
        A.copy_(dev(Ah))
        f.project(A, B, X, Q)
        launches.append(f.last_launch_count)
        assert rel(host(Q), oracle.project(Ah, P.B, Xh, z, w)) <= TOL, it
    assert len(set(launches)) == 1   # the replayed graph holds the same kernels


@pytest.mark.parametrize("rule,n_e,aspect,n", [(synth.RULE_TRAPEZOID, 16, 1.0, 260),
                                               (synth.RULE_TRAPEZOID_ENDPOINT, 8, 1.0, 200),
                                               (synth.RULE_GAUSS_LEGENDRE, 6, 0.5, 132)])
def test_real_pencil_mode_parity(rule, n_e, aspect, n):
    """NEXT-2b: real A, B and a contour symmetric about the real axis — each conjugate pole pair
    is factored once with [R | conj R]; Q and Q_L must still equal the oracle's per-node sums.
    The endpoint rule has real poles (single units)."""
    P = synth.make_pencil("R2", n=n, m0=21)
    s = P.spec
    z, w = oracle.nodes(s.c, s.r, aspect, n_e, rule)
    f = Feast(P.n, P.m0, s.c, s.r, aspect, n_e, rule, fb.BI, False, real_pencil=True)
    zz, _, j0, j1 = f.nodes()
    n_real = sum(1 for x in zz if abs(x.imag) < 1e-12)
    assert j1 - j0 == (len(zz) - n_real) // 2 + n_real          # one unit per orbit
    A, B, X = dev(P.A), dev(P.B), dev(P.X0)
    Vin = synth.random_block(P.n, P.m0, 7)
    Q = host(f.project(A, B, X))
    assert rel(Q, oracle.project(P.A, P.B, P.X0, z, w)) <= TOL
    Qb, QLb = f.project_bi(A, B, X, dev(Vin))
    assert rel(host(Qb), oracle.project(P.A, P.B, P.X0, z, w)) <= TOL
    assert rel(host(QLb), oracle.project(P.A, P.B, Vin, z, w, left=True)) <= TOL
    stats, worst = f.node_stats()
    assert all(v > 0 for v in stats) and 0 <= worst < len(zz)   # every node (both poles) reported


def test_real_pencil_mode_full_size_and_guards():
    """R2 at full size (n = 2048): parity, half the factorisation units; a complex A is refused
    at run time (device check) and a contour off the real axis at set-up."""
    P = synth.make_pencil("R2")
    s = P.spec
    z, w = _oracle_nodes(P)
    f = _handle(P, real_pencil=True)
    _, _, j0, j1 = f.nodes()
    assert j1 - j0 == P.q // 2
    Q = host(f.project(dev(P.A), dev(P.B), dev(P.X0)))
    assert rel(Q, oracle.project(P.A, P.B, P.X0, z, w)) <= TOL
    x = (P.lam - s.c) / s.r
    Qs = P.V @ ((1 / (1 + x ** P.q))[:, None] * np.linalg.solve(P.V, P.X0))
    assert rel(Q, Qs) <= TOL
    Ac = dev(P.A + 1e-3j * np.eye(P.n))
    with pytest.raises(FeastError, match="imaginary"):
        f.project(Ac, dev(P.B), dev(P.X0))
    with pytest.raises(FeastError):
        Feast(P.n, P.m0, 0.2 + 0.1j, s.r, s.aspect, s.n_e, s.rule, fb.RIGHT, False, real_pencil=True)


@pytest.mark.parametrize("n,m0", [(160, 12), (300, 25)])
def test_complex_symmetric_bi_parity(n, m0):
    """NEXT-2a: C3-recipe (complex-symmetric) pencil in a Bi handle with the complex-symmetric
    mode: the left block is computed by right solves of conj(B^H V); Q and Q_L match the oracle
    (which runs the conjugate-transposed substitution), for project_bi and project_left."""
    P = synth.make_pencil("C3", n=n, m0=m0)
    assert np.abs(P.A - P.A.T).max() == 0 and np.abs(P.B - P.B.T).max() == 0
    z, w = _oracle_nodes(P)
    Vin = synth.random_block(P.n, P.m0, 3)
    f = _handle(P, mode=fb.BI, complex_symmetric=True)
    A, B = dev(P.A), dev(P.B)
    Q, QL = f.project_bi(A, B, dev(P.X0), dev(Vin))
    assert rel(host(Q), oracle.project(P.A, P.B, P.X0, z, w)) <= TOL
    assert rel(host(QL), oracle.project(P.A, P.B, Vin, z, w, left=True)) <= TOL
    QL2 = f.project_left(A, B, dev(Vin))
    assert rel(host(QL2), oracle.project(P.A, P.B, Vin, z, w, left=True)) <= TOL
    Q2 = f.project(A, B, dev(P.X0))
    assert rel(host(Q2), oracle.project(P.A, P.B, P.X0, z, w)) <= TOL


def test_count_estimate():
    """NEXT-3: feast_estimate_count = Re tr(U^H rho(B^-1 A) U) / m0.  U = I (m0 = n) gives
    m0 * estimate = Re sum rho(lambda_i) exactly (closed form from the known spectrum); a random U
    matches the oracle's estimate, and at C2 size the estimate lands near the true count."""
    P = synth.make_pencil("C1", n=96, m0=96)
    f = _handle(P)
    est, _ = f.estimate_count(dev(P.A), dev(P.B), dev(np.eye(P.n, dtype=complex)))
    x = (P.lam - P.spec.c) / P.spec.r
    exact = float(np.sum(1 / (1 + x ** P.q)).real)
    assert abs(est * P.m0 - exact) <= 1e-10 * max(1.0, abs(exact))
    P = synth.make_pencil("C2", n=300, m0=40)
    z, w = _oracle_nodes(P)
    f = _handle(P)
    U = synth.random_block(P.n, P.m0, 77)
    est, Q = f.estimate_count(dev(P.A), dev(P.B), dev(U))
    Qo = oracle.project(P.A, P.B, U, z, w)
    assert rel(host(Q), Qo) <= TOL
    assert abs(est - float(np.trace(U.conj().T @ Qo).real) / P.m0) <= 1e-10 * max(1.0, abs(est))
    P = synth.make_pencil("C2")
    f = _handle(P)
    est, _ = f.estimate_count(dev(P.A), dev(P.B), dev(P.X0))
    true_m = int(np.sum(np.abs(P.lam - P.spec.c) < P.spec.r))
    assert abs(est - true_m) <= 0.25 * true_m, (est, true_m)


@pytest.mark.parametrize("segs,K,rule", [
    ([("line", -0.4 - 0.4j, 0.4 - 0.4j), ("line", 0.4 - 0.4j, 0.4 + 0.4j), ("line", 0.4 + 0.4j, -0.4 + 0.4j),
      ("line", -0.4 + 0.4j, -0.4 - 0.4j)], 8, synth.RULE_TRAPEZOID),
    ([("arc", 0.0, 0.5, 0.0, np.pi), ("line", -0.5, 0.5)], 8, synth.RULE_GAUSS_LEGENDRE)])
def test_composite_contour_projector(segs, K, rule):
    """NEXT-4: square / semicircle contours glued from segments; Q matches the oracle
    with the oracle's own contour nodes, and the spectral identity with rho evaluated by the oracle."""
    P = synth.make_pencil("C1", n=150, m0=20)
    zo, wo = oracle.contour_nodes(segs, K, rule)
    f = Feast(P.n, P.m0, 0j, 1.0, 1.0, 8, 0, fb.RIGHT, True, segments=segs, k_per_segment=K, segment_rule=rule)
    Q = host(f.project(dev(P.A), None, dev(P.X0)))
    assert rel(Q, oracle.project(P.A, None, P.X0, zo, wo)) <= TOL
    Qs = P.V @ (oracle.rho(zo, wo, P.lam)[:, None] * np.linalg.solve(P.V, P.X0))
    assert rel(Q, Qs) <= TOL
    assert np.max(np.abs(f.filter(P.lam[:5]) - oracle.rho(zo, wo, P.lam[:5]))) < 1e-12


def test_row_sharded_reduce_partials():
    """a7 row-sharded over ranks: each virtual rank's m0 x m0 partial
    (rows [r n/P, (r+1) n/P) of A Q and B Q) is handed to the all-reduce callback; the partials
    of all ranks sum to QL^H A Q and QL^H B Q (checked against the unsharded product)."""
    import ctypes
    P = synth.make_pencil("C2", n=230, m0=18)
    world = 4                # q = 16 nodes over 4 ranks; 230 rows split 57/58 (ragged)
    A, B, Q = dev(P.A), dev(P.B), dev(synth.random_block(P.n, P.m0, 5))
    full = _handle(P)
    Ah, Bh = full.reduce(A, B, Q)
    Ah, Bh = host(Ah), host(Bh)
    got = {"A": 0, "B": 0}
    for r in range(world):
        f = _handle(P, rank=r, world=world, partial=True)
        seen = []

        def cb(buf, count, stream, user, seen=seen):
            torch.cuda.synchronize()
            t = torch.as_tensor(fb._CudaPtr(buf, count), device="cuda")
            seen.append(t.clone().view(torch.complex128).cpu().numpy())
            return 0

        f._ar = fb.ALLREDUCE_FN(cb)
        assert f.lib.feast_set_allreduce(f.h, f._ar, None) == 0
        pa, pb = f.reduce(A, B, Q)
        assert len(seen) == 2   # Ahat, Bhat partials (ld = m0: one call each)
        got["A"] = got["A"] + seen[0].reshape(P.m0, P.m0).T
        got["B"] = got["B"] + seen[1].reshape(P.m0, P.m0).T
    assert rel(got["A"], Ah) <= 1e-12 and rel(got["B"], Bh) <= 1e-12


def test_row_sharded_rhs_partials():
    """a1 row-sharded over ranks: rank r forms rows [r n/P, (r+1) n/P) of R = B X (zeros
    elsewhere) and hands the block to the all-reduce callback, whose sum over ranks must be B X."""
    P = synth.make_pencil("C2", n=230, m0=18)
    world = 4
    A, B, X = dev(P.A), dev(P.B), dev(P.X0)
    total = 0
    for r in range(world):
        f = _handle(P, rank=r, world=world, partial=True)
        seen = []

        def cb(buf, count, stream, user, seen=seen):
            torch.cuda.synchronize()
            t = torch.as_tensor(fb._CudaPtr(buf, count), device="cuda")
            seen.append(t.clone().view(torch.complex128).cpu().numpy())
            return 0

        f._ar = fb.ALLREDUCE_FN(cb)
        assert f.lib.feast_set_allreduce(f.h, f._ar, None) == 0
        f.project(A, B, X)
        ld = seen[0].size // P.m0
        part = seen[0].reshape(P.m0, ld).T[:P.n]
        r0, r1 = r * P.n // world, (r + 1) * P.n // world
        assert np.all(part[:r0] == 0) and np.all(part[r1:] == 0)
        total = total + part
    assert rel(total, P.B @ P.X0) <= 1e-13


@pytest.mark.parametrize("key,n,m0", [("C2", 300, 20), ("C3", 700, 24), ("C3", 1300, 9)])
def test_row_swap_variants_bit_identical(monkeypatch, key, n, m0):
    """Row swaps are pure data movement: the default coalesced kernel (slot-traced gather/scatter),
    the per-column swap chain (FEAST_LASWP=chain), the per-CTA permutation kernel
    (FEAST_LASWP=perm), the panels' swaps done by a separate launch instead of inside the panel
    kernel (FEAST_PANEL_SWAP=0) and the L-column swaps on the main stream instead of the side
    stream (FEAST_LSWAP_SIDE=0) must give BIT-identical projectors, equal to the oracle's.  The C3 recipe
    (random symmetric H + iD) pivots off the diagonal in most columns, so every swap path moves
    rows; n = 1300 has ragged panels and several cluster sizes."""
    P = synth.make_pencil(key, n=n, m0=m0)
    z, w = _oracle_nodes(P)
    out = {}
    for v in ("coalesced", "chain", "perm", "unfused", "lswap_main"):
        monkeypatch.setenv("FEAST_LASWP", v if v in ("coalesced", "chain", "perm") else "coalesced")
        monkeypatch.setenv("FEAST_PANEL_SWAP", "0" if v == "unfused" else "1")
        monkeypatch.setenv("FEAST_LSWAP_SIDE", "0" if v == "lswap_main" else "1")
        f = _handle(P)
        out[v] = host(f.project(dev(P.A), dev(P.B), dev(P.X0)))
        f.project(dev(P.A), dev(P.B), dev(P.X0))   # graph capture of the multi-stream sequence
    for v in ("chain", "perm", "unfused", "lswap_main"):
        assert np.array_equal(out["coalesced"], out[v]), v
    assert rel(out["coalesced"], oracle.project(P.A, P.B, P.X0, z, w)) <= TOL


@pytest.mark.parametrize("one_row", ["0", "1"])
def test_panel_thread_layouts(monkeypatch, one_row):
    """Both panel thread layouts for 129..256 rows per CTA (128 threads x 2 rows, the default for
    many concurrent nodes; 256 threads x 1 row, the default for <= 4) give the oracle's projector
    on heights that walk through cluster sizes 8 -> 1 (n = 1100, ragged)."""
    monkeypatch.setenv("FEAST_PANEL_1ROW", one_row)
    P = synth.make_pencil("C2", n=1100, m0=12)
    z, w = _oracle_nodes(P)
    f = _handle(P)
    Q = host(f.project(dev(P.A), dev(P.B), dev(P.X0)))
    assert rel(Q, oracle.project(P.A, P.B, P.X0, z, w)) <= TOL


@pytest.mark.parametrize("key,n,m0", [("C2", 220, 24), ("C4", 200, 30)])
def test_projector_parity_at_later_iterations(key, n, m0):
    """Parity protocol P1 at k > 1: the GPU projector applied to the ORACLE's
    iterate X^(k-1) (after two oracle R-FEAST iterations) matches the oracle's projector."""
    P = synth.make_pencil(key, n=n, m0=m0)
    s = P.spec
    z, w = _oracle_nodes(P)
    X = P.X0
    for _ in range(2):
        X = oracle.feast_iterate(P.A, P.B, X, None, z, w, s.c, s.r, s.aspect)["X"]
    f = _handle(P)
    Q = host(f.project(dev(P.A), dev(P.B), dev(X)))
    assert rel(Q, oracle.project(P.A, P.B, X, z, w)) <= TOL


def test_worst_pivot_node_solution():
    """Parity protocol P2: the per-node solve Y_j = (z_j B - A)^-1 B X of the node with the
    smallest pivot ratio (feast_node_stats), isolated as a one-node virtual rank (its partial is
    w_j Y_j), matches the oracle's naive-LU solve of that node."""
    P = synth.make_pencil("C2", n=240, m0=12)
    z, w = _oracle_nodes(P)
    f = _handle(P)
    f.project(dev(P.A), dev(P.B), dev(P.X0))
    stats, worst = f.node_stats()
    assert worst == int(np.argmin(stats))
    g = _handle(P, rank=worst, world=P.q, partial=True)                      # owns exactly node `worst`
    part = host(g.project(dev(P.A), dev(P.B), dev(P.X0)))
    Yj = part / w[worst]
    Yo = oracle.project(P.A, P.B, P.X0, z, np.ones_like(w), worst, worst + 1)
    assert rel(Yj, Yo) <= TOL


@pytest.mark.parametrize("n,m0", [(257, 9), (513, 17), (1000, 31), (2049, 8)])
def test_ragged_sizes_across_panel_paths(n, m0):
    """Heights around the panel-kernel boundaries: 1 -> 2 -> 4 -> 8 -> 16 CTAs per cluster as
    L = n - k falls (256 rows per CTA), ragged last blocks; oracle parity."""
    P = synth.make_pencil("C2", n=n, m0=m0)
    z, w = _oracle_nodes(P)
    f = _handle(P)
    Q = host(f.project(dev(P.A), dev(P.B), dev(P.X0)))
    assert rel(Q, oracle.project(P.A, P.B, P.X0, z, w)) <= TOL


@pytest.mark.parametrize("n", [4200, 8400])
def test_register_panel_height_spectral(n):
    """Tall panels: n = 4200 > 16 x 256 rows starts on the 256-thread shared-memory cluster
    kernel (two rows per thread, 263 rows per CTA); n = 8400 > 16 x 512 on the register-chunk
    kernel, both handing over to the 128-thread kernels as L = n - k falls; checked with the
    spectral identity (closed-form filter)."""
    P = synth.make_pencil_torch("C2", n=n, m0=16)
    s = P.spec
    f = _handle(P)
    Q = f.project(P.A, P.B, P.X0)
    rho = 1.0 / (1.0 + ((P.lam - s.c) / s.r) ** P.q)
    Qs = P.V @ (rho[:, None] * torch.linalg.solve(P.V, P.X0))
    assert float(torch.linalg.norm(Q - Qs) / torch.linalg.norm(Qs)) <= TOL


@pytest.mark.parametrize("vtall", ["1", "0"])
def test_very_tall_panels(monkeypatch, vtall):
    """Panels of 1025..2048 rows per CTA (C5's first half at n = 32768) on the cluster kernel
    (FEAST_VTALL=1: 8-wide panels, 256 threads x 8 rows) or on the register-chunk kernel: with
    clusters capped at 8 CTAs, n = 8400 starts at 1050 rows per CTA and walks every panel regime
    down to one CTA; spectral identity with the closed-form filter."""
    monkeypatch.setenv("FEAST_VTALL", vtall)
    monkeypatch.setenv("FEAST_CS_MAX", "8")
    P = synth.make_pencil_torch("C2", n=8400, m0=16)
    s = P.spec
    f = _handle(P)
    Q = f.project(P.A, P.B, P.X0)
    rho = 1.0 / (1.0 + ((P.lam - s.c) / s.r) ** P.q)
    Qs = P.V @ (rho[:, None] * torch.linalg.solve(P.V, P.X0))
    assert float(torch.linalg.norm(Q - Qs) / torch.linalg.norm(Qs)) <= TOL


@pytest.mark.parametrize("variant", ["4", "5", "2"])
def test_tall_panel_variants(monkeypatch, variant):
    """The 513..1024-rows-per-CTA cluster panels (n = 8400: 525 rows per CTA at the start):
    256 threads x 4 rows with an 8-column register chunk (4, default), with a 4-column chunk and
    12 shared-memory columns (5), 512 threads x 2 rows (2) — each gives the spectral projector."""
    monkeypatch.setenv("FEAST_TALL_VARIANT", variant)
    P = synth.make_pencil_torch("C2", n=8400, m0=16)
    s = P.spec
    f = _handle(P)
    Q = f.project(P.A, P.B, P.X0)
    rho = 1.0 / (1.0 + ((P.lam - s.c) / s.r) ** P.q)
    Qs = P.V @ (rho[:, None] * torch.linalg.solve(P.V, P.X0))
    assert float(torch.linalg.norm(Q - Qs) / torch.linalg.norm(Qs)) <= TOL


@pytest.mark.parametrize("btrsm", ["1", "0"])
@pytest.mark.parametrize("nb", ["64", "128", "256", "512"])
@pytest.mark.parametrize("n,m0", [(1000, 24), (1345, 8)])
def test_two_level_substitutions(monkeypatch, btrsm, nb, n, m0):
    """Back substitution, left solves and (factor cache) forward substitution with outer blocks of
    FEAST_SOLVE_NB rows (64 = the one-level sweep; 512 = two fused 256-row block solves coupled by
    a GEMM), with the fused DMMA block solve (btrsm) or the one-level launch chain: right and left
    projectors from one LU, and the cached-factor path, equal the oracle's on ragged sizes (n not a
    multiple of 64 or of the outer block)."""
    monkeypatch.setenv("FEAST_SOLVE_NB", nb)
    monkeypatch.setenv("FEAST_BTRSM", btrsm)
    P = synth.make_pencil("C4", n=n, m0=m0)
    z, w = _oracle_nodes(P)
    V = synth.random_block(n, m0, 17)
    f = _handle(P, fb.BI)
    Q, QL = f.project_bi(dev(P.A), None, dev(P.X0), dev(V))
    assert rel(host(Q), oracle.project(P.A, None, P.X0, z, w)) <= TOL
    assert rel(host(QL), oracle.project(P.A, None, V, z, w, left=True)) <= TOL
    g = _handle(P)
    g.factor_cache(True)
    A, X = dev(P.A), dev(P.X0)
    g.project(A, None, X)
    Q2 = host(g.project(A, None, X))          # substitution-only call on the cached factors
    assert rel(Q2, oracle.project(P.A, None, P.X0, z, w)) <= TOL


def test_async_mode_pipelines_and_defers_status():
    """feast_set_async: projector and reduce calls return once enqueued; results (read in stream
    order) equal the oracle's; the singular-node status of a projection is reported by
    feast_sync instead of the call."""
    P = synth.make_pencil("C2", n=260, m0=12)
    z, w = _oracle_nodes(P)
    f = _handle(P)
    f.set_async(True)
    A, B = dev(P.A), dev(P.B)
    X2 = synth.random_block(P.n, P.m0, 23)
    Q1 = f.project(A, B, dev(P.X0))
    Q2 = f.project(A, B, dev(X2))
    Ah, Bh = f.reduce(A, B, Q2)
    assert f.sync() == fb.OK
    assert rel(host(Q1), oracle.project(P.A, P.B, P.X0, z, w)) <= TOL
    Q2o = oracle.project(P.A, P.B, X2, z, w)
    assert rel(host(Q2), Q2o) <= TOL
    assert rel(host(Ah), Q2o.conj().T @ P.A @ Q2o) <= 1e-10
    # singular node: the call returns, feast_sync reports it
    p = np.exp(1j * np.pi / 4)
    Ad = np.diag([p, 0.1, 3.0, -0.2 + 0.1j]).astype(complex)
    g = Feast(4, 2, 0j, 1.0, 1.0, 4, fb.RULE_TRAPEZOID, fb.RIGHT, True)
    zz, _, _, _ = g.nodes()
    Ad[0, 0] = zz[0]
    g.set_async(True)
    g.project(dev(Ad), None, dev(np.eye(4)[:, :2]))
    with pytest.raises(FeastError) as e:
        g.sync()
    assert e.value.code == fb.E_SINGULAR


@pytest.mark.parametrize("nbo", ["256", "512", "1024"])
@pytest.mark.parametrize("btrsm", ["1", "0"])
def test_outer_block_sizes(monkeypatch, nbo, btrsm):
    """LU outer blocks of FEAST_NBO columns (U12 = L11^-1 A12 by the fused block solve in 256-row
    pieces, or the one-level chain), ragged n, right and left projectors vs the oracle."""
    monkeypatch.setenv("FEAST_NBO", nbo)
    monkeypatch.setenv("FEAST_BTRSM", btrsm)
    P = synth.make_pencil("C2", n=1100, m0=10)
    z, w = _oracle_nodes(P)
    V = synth.random_block(P.n, P.m0, 31)
    f = _handle(P, fb.BI)
    Q, QL = f.project_bi(dev(P.A), dev(P.B), dev(P.X0), dev(V))
    assert rel(host(Q), oracle.project(P.A, P.B, P.X0, z, w)) <= TOL
    assert rel(host(QL), oracle.project(P.A, P.B, V, z, w, left=True)) <= TOL


@pytest.mark.parametrize("join", ["1", "0"])
def test_substitution_join_modes(monkeypatch, join):
    """Substitutions once over the whole batch after joining the node groups (default) or per
    group (FEAST_SUBST_JOIN=0): right + left projectors and the cached-factor path vs the oracle."""
    monkeypatch.setenv("FEAST_SUBST_JOIN", join)
    P = synth.make_pencil("C4", n=520, m0=12)
    z, w = _oracle_nodes(P)
    V = synth.random_block(P.n, P.m0, 41)
    f = _handle(P, fb.BI)
    Q, QL = f.project_bi(dev(P.A), None, dev(P.X0), dev(V))
    assert rel(host(Q), oracle.project(P.A, None, P.X0, z, w)) <= TOL
    assert rel(host(QL), oracle.project(P.A, None, V, z, w, left=True)) <= TOL
    g = _handle(P)
    g.factor_cache(True)
    A, X = dev(P.A), dev(P.X0)
    g.project(A, None, X)
    assert rel(host(g.project(A, None, X)), oracle.project(P.A, None, P.X0, z, w)) <= TOL


def test_workspace_query_after_bind_keeps_layout():
    """feast_workspace_bytes after feast_bind_workspace only reports the size: the bound layout,
    the batch and a captured graph stay valid (it used to null the workspace pointers)."""
    import ctypes
    P = synth.make_pencil("C2", n=300, m0=16)
    z, w = _oracle_nodes(P)
    f = _handle(P)
    A, B, X = dev(P.A), dev(P.B), dev(P.X0)
    Q = f.project(A, B, X)
    f.project(A, B, X, Q)                     # second identical call: captured into a graph
    nb = ctypes.c_size_t()
    assert f.lib.feast_workspace_bytes(f.h, ctypes.byref(nb)) == 0
    assert nb.value <= f.workspace.numel()
    Q2 = host(f.project(A, B, X, Q))          # graph replay on the same layout
    assert rel(Q2, oracle.project(P.A, P.B, P.X0, z, w)) <= TOL


@pytest.mark.parametrize("stagger", ["1", "2", "5"])
def test_staggered_node_groups(monkeypatch, stagger):
    """FEAST_STAGGER = d: node group g starts after group g - 1 finished d outer LU steps (the
    groups' latency-bound tails overlap other groups' GEMMs); d larger than the number of steps
    degenerates to sequential groups.  Right + left projectors vs the oracle, and a repeated call
    (graph capture / replay of the event dependencies)."""
    monkeypatch.setenv("FEAST_STAGGER", stagger)
    P = synth.make_pencil("C2", n=700, m0=12)
    z, w = _oracle_nodes(P)
    V = synth.random_block(P.n, P.m0, 43)
    f = _handle(P, fb.BI)
    A, B, X, Vd = dev(P.A), dev(P.B), dev(P.X0), dev(V)
    Qo, QLo = oracle.project(P.A, P.B, P.X0, z, w), oracle.project(P.A, P.B, V, z, w, left=True)
    for _ in range(3):
        Q, QL = f.project_bi(A, B, X, Vd)
        assert rel(host(Q), Qo) <= TOL and rel(host(QL), QLo) <= TOL


def test_binding_rejects_wrong_column_counts():
    """The library reads / writes exactly n columns of A, B and m0 of X, V, Q, QL: the binding
    refuses a block with another column count instead of letting the kernels run past it."""
    P = synth.make_pencil("C2", n=64, m0=8)
    f = _handle(P)
    A, B, X = dev(P.A), dev(P.B), dev(P.X0)
    for bad in (lambda: f.project(A, B, X[:, :7]), lambda: f.project(A[:, :63], B, X),
                lambda: f.project(A, B, X, dev(np.zeros((P.n, 9), complex)))):
        with pytest.raises(FeastError) as e:
            bad()
        assert e.value.code == fb.E_ARG


@pytest.mark.parametrize("key,n,m0", [("C2", 700, 24), ("C4", 600, 40)])
def test_substitution_dot_form(monkeypatch, key, n, m0):
    """FEAST_SUBST_DOT=1: every substitution (right back, left U^H / L^H, the cached forward
    solve) in dot form — each 256-row outer block takes all solved rows' contribution in one
    long-K GEMM before its diagonal block — gives the oracle's Q (and Q_L; with cached factors
    too) on heights of several ragged outer blocks, and agrees with the right-looking form to
    rounding."""
    P = synth.make_pencil(key, n=n, m0=m0)
    z, w = _oracle_nodes(P)
    A, B, X = dev(P.A), dev(P.B), dev(P.X0)
    out = {}
    for v in ("0", "1"):
        monkeypatch.setenv("FEAST_SUBST_DOT", v)
        f = _handle(P, mode=fb.BI)
        f.factor_cache(True)
        Q, QL = f.project_bi(A, B, X, X)
        X2 = dev(synth.random_block(P.n, P.m0, 7))
        Qc = f.project(A, B, X2)              # cached factors: forward + back substitution only
        out[v] = (host(Q), host(QL), host(Qc))
    Qo = oracle.project(P.A, P.B, P.X0, z, w)
    QLo = oracle.project(P.A, P.B, P.X0, z, w, left=True)
    Qco = oracle.project(P.A, P.B, synth.random_block(P.n, P.m0, 7), z, w)
    for (Q, QL, Qc) in out.values():
        assert rel(Q, Qo) <= TOL and rel(QL, QLo) <= TOL and rel(Qc, Qco) <= TOL
    for a, b in zip(out["0"], out["1"]):
        assert rel(a, b) <= 1e-12


@pytest.mark.parametrize("key,n,m0", [("C2", 700, 24), ("C4", 600, 40)])
def test_outer_u12_dot_form(monkeypatch, key, n, m0):
    """FEAST_U12_DOT=2: the outer blocks' U12 = L11^-1 A12 in dot form (each 64-row block takes
    the solved blocks' contribution in one GEMM with K = 64 i, then its 64x64 inverse) gives the
    oracle's Q and Q_L on heights of several ragged outer blocks (augmented columns included),
    and agrees with the right-looking form (FEAST_U12_DOT=0) to rounding."""
    P = synth.make_pencil(key, n=n, m0=m0)
    z, w = _oracle_nodes(P)
    A, B, X = dev(P.A), dev(P.B), dev(P.X0)
    out = {}
    for v in ("0", "2"):
        monkeypatch.setenv("FEAST_U12_DOT", v)
        f = _handle(P, mode=fb.BI)
        Q, QL = f.project_bi(A, B, X, X)
        out[v] = (host(Q), host(QL))
    Qo = oracle.project(P.A, P.B, P.X0, z, w)
    QLo = oracle.project(P.A, P.B, P.X0, z, w, left=True)
    for (Q, QL) in out.values():
        assert rel(Q, Qo) <= TOL and rel(QL, QLo) <= TOL
    for a, b in zip(out["0"], out["2"]):
        assert rel(a, b) <= 1e-12


@pytest.mark.parametrize("outer", ["0", "1"])
def test_substitution_inner_dot_form(monkeypatch, outer):
    """FEAST_SUBST_INNER_DOT=2: the 64-row blocks inside every substitution outer block (right
    back, left U^H / L^H, the cached forward solve) in dot form, with right-looking (0) or dot-form
    (1) outer blocks: the oracle's Q, Q_L and cached-factor Q on several ragged outer blocks, and
    the right-looking inner form's results to rounding."""
    P = synth.make_pencil("C4", n=600, m0=40)
    z, w = _oracle_nodes(P)
    A, B, X = dev(P.A), dev(P.B), dev(P.X0)
    X2 = synth.random_block(P.n, P.m0, 7)
    monkeypatch.setenv("FEAST_SUBST_DOT", outer)
    out = {}
    for v in ("0", "2"):
        monkeypatch.setenv("FEAST_SUBST_INNER_DOT", v)
        f = _handle(P, mode=fb.BI)
        f.factor_cache(True)
        Q, QL = f.project_bi(A, B, X, X)
        Qc = f.project(A, B, dev(X2))
        out[v] = (host(Q), host(QL), host(Qc))
    Qo = oracle.project(P.A, P.B, P.X0, z, w)
    QLo = oracle.project(P.A, P.B, P.X0, z, w, left=True)
    Qco = oracle.project(P.A, P.B, X2, z, w)
    for (Q, QL, Qc) in out.values():
        assert rel(Q, Qo) <= TOL and rel(QL, QLo) <= TOL and rel(Qc, Qco) <= TOL
    for a, b in zip(out["0"], out["2"]):
        assert rel(a, b) <= 1e-12
