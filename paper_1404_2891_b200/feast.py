"""Thin Python binding of the C ABI in include/feast.h (argument marshalling only).

Every step of the FEAST hot path runs in libfeast_b200.so's sm_100a kernels; PyTorch only
provides device memory, the CUDA stream and torch.distributed: the library calls back into
torch.distributed.all_reduce for the cross-rank node sum and the row-sharded
assemblies, on its own stream.  There is no CPU fallback: if the library is missing this
module raises.

Matrices are complex128 COLUMN-MAJOR CUDA tensors (stride(0) == 1, stride(1) = ld >= rows),
e.g. ``colmajor(torch.from_numpy(np.asfortranarray(a)))`` or ``empty_colmajor(n, m)``.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfeast_b200.so")

RULE_TRAPEZOID = 0
RULE_TRAPEZOID_ENDPOINT = 1
RULE_GAUSS_LEGENDRE = 2
RIGHT = 0
BI = 1

OK, E_ARG, E_NOMEM, E_SINGULAR, E_CUDA, E_COMM, E_STATE, E_REDUCED, W_ILLCOND = 0, -1, -2, -3, -4, -5, -6, -7, 1
_NAMES = {E_ARG: "FEAST_E_ARG", E_NOMEM: "FEAST_E_NOMEM", E_SINGULAR: "FEAST_E_SINGULAR", E_CUDA: "FEAST_E_CUDA",
          E_COMM: "FEAST_E_COMM", E_STATE: "FEAST_E_STATE", E_REDUCED: "FEAST_E_REDUCED"}

ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p)

# every symbol include/feast.h declares (checked by tests/test_abi.py)
EXPORTS = ["feast_init", "feast_workspace_bytes", "feast_bind_workspace", "feast_nodes", "feast_project",
           "feast_project_left", "feast_project_bi", "feast_reduce", "feast_set_allreduce", "feast_set_partial",
           "feast_iterate",
           "feast_node_stats", "feast_factor_cache", "feast_set_real_pencil",
           "feast_set_complex_symmetric", "feast_estimate_count", "feast_set_contour", "feast_filter",
           "feast_estimate_count_bi", "feast_set_count_estimate", "feast_monitors", "feast_filter_gap",
           "feast_set_async", "feast_sync",
           "feast_last_launch_count", "feast_profile", "feast_profile_summary",
           "feast_profile_records", "feast_last_error",
           "feast_version", "feast_destroy"]
K_CLASSES = ["shift", "panel", "laswp", "trsm", "zgemm", "perm", "accum", "other"]


class FeastError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{_NAMES.get(code, code)}: {msg}")
        self.code = code


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libfeast_b200.so (raises if it was not built: no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not built; run `python -m paper_1404_2891_b200.build` (no CPU fallback)")
    lib = ctypes.CDLL(path)
    P, I64, I32, D, SZ = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double, ctypes.c_size_t
    lib.feast_init.argtypes = [ctypes.POINTER(P), I64, I64, D, D, D, D, I32, I32, I32, I32, I32, I32, I32, P]
    lib.feast_workspace_bytes.argtypes = [P, ctypes.POINTER(SZ)]
    lib.feast_bind_workspace.argtypes = [P, P, SZ]
    lib.feast_nodes.argtypes = [P, P, P, P, P, P]
    lib.feast_project.argtypes = [P, P, I64, P, I64, P, I64, P, I64]
    lib.feast_project_left.argtypes = [P, P, I64, P, I64, P, I64, P, I64]
    lib.feast_project_bi.argtypes = [P, P, I64, P, I64, P, I64, P, I64, P, I64, P, I64]
    lib.feast_reduce.argtypes = [P, P, I64, P, I64, P, I64, P, I64, P, I64, P, I64]
    lib.feast_set_allreduce.argtypes = [P, ALLREDUCE_FN, P]
    lib.feast_set_partial.argtypes = [P, I32]
    lib.feast_iterate.argtypes = [P, P, I64, P, I64, P, I64, P, I64, P, P, P]
    lib.feast_node_stats.argtypes = [P, P, P]
    lib.feast_last_launch_count.argtypes = [P]
    lib.feast_last_launch_count.restype = I64
    lib.feast_factor_cache.argtypes = [P, I32]
    lib.feast_set_real_pencil.argtypes = [P, I32]
    lib.feast_set_complex_symmetric.argtypes = [P, I32]
    lib.feast_estimate_count.argtypes = [P, P, I64, P, I64, P, I64, P, I64, P]
    lib.feast_set_contour.argtypes = [P, I32, P, P, I32, I32]
    lib.feast_filter.argtypes = [P, I64, P, P]
    lib.feast_estimate_count_bi.argtypes = [P, P, I64, P, I64, P, I64, P, I64, P, I64, P, I64, P, P]
    lib.feast_set_count_estimate.argtypes = [P, I32]
    lib.feast_set_async.argtypes = [P, I32]
    lib.feast_sync.argtypes = [P]
    lib.feast_monitors.argtypes = [P, P, P, P, P, P]
    lib.feast_filter_gap.argtypes = [P, I64, P, I64, P, P, P, P, P, P]
    lib.feast_profile.argtypes = [P, I32]
    lib.feast_profile_summary.argtypes = [P, I32, P, P, P, P]
    lib.feast_profile_records.argtypes = [P, I64, P, P, P, P, P, P]
    lib.feast_last_error.argtypes = [P]
    lib.feast_last_error.restype = ctypes.c_char_p
    lib.feast_version.restype = ctypes.c_char_p
    lib.feast_destroy.argtypes = [P]
    lib.feast_destroy.restype = None
    _lib = lib
    return lib


def colmajor(t: torch.Tensor) -> torch.Tensor:
    """Column-major copy of a 2-D tensor (complex128 kept)."""
    return t.t().contiguous().t()


def empty_colmajor(rows: int, cols: int, device="cuda", dtype=torch.complex128) -> torch.Tensor:
    return torch.empty((cols, rows), dtype=dtype, device=device).t()


def _ptr_ld(t, rows, name, device=None, cols=None):
    if t is None:
        return None, 0
    if t.dtype != torch.complex128 or not t.is_cuda or t.dim() != 2:
        raise FeastError(E_ARG, f"{name} must be a 2-D complex128 CUDA tensor")
    if device is not None and t.device != device:
        raise FeastError(E_ARG, f"{name} is on {t.device}, the handle on {device}")
    if t.shape[0] != rows or (rows > 1 and t.stride(0) != 1):
        raise FeastError(E_ARG, f"{name} must be column-major with {rows} rows")
    if cols is not None and t.shape[1] != cols:   # the library reads / writes exactly `cols` columns
        raise FeastError(E_ARG, f"{name} must have {cols} columns (has {t.shape[1]})")
    ld = t.stride(1) if t.shape[1] > 1 else max(rows, 1)
    if ld < rows:
        raise FeastError(E_ARG, f"{name}: leading dimension {ld} < {rows} rows")
    return ctypes.c_void_p(t.data_ptr()), ld


def _dist_world(group=None) -> int:
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group)
    return 1


def make_allreduce_callback(device, group=None):
    """The feast_allreduce_fn the library calls for every cross-rank sum (the node sum of Q / QL,
    the row-sharded a1 / a7 assemblies, the residual norms): SUM all-reduce of `count` float64
    values at the raw pointer `buf`, in place, ordered on the library's stream.  The library
    always passes one contiguous flat block (it packs Q and QL itself), so no tensor layout is
    involved here.  `device` is the torch device of the buffers (cuda:k; "cpu" wraps a host
    pointer — the CPU tests of this marshalling with gloo)."""
    import torch.distributed as dist
    device = torch.device(device)

    def cb(buf, count, stream, user):
        try:
            if device.type == "cuda":
                t = torch.as_tensor(_CudaPtr(buf, count), device=device)
                with torch.cuda.stream(torch.cuda.ExternalStream(stream, device=device)):
                    dist.all_reduce(t, group=group)   # enqueued on the library's stream
            else:
                import numpy as np
                arr = np.ctypeslib.as_array(ctypes.cast(buf, ctypes.POINTER(ctypes.c_double)), shape=(int(count),))
                dist.all_reduce(torch.from_numpy(arr), group=group)
            return 0
        except Exception:  # noqa: BLE001 — reported as FEAST_E_COMM by the library
            return 1

    return cb


class _CudaPtr:
    """__cuda_array_interface__ shim so the all-reduce callback can wrap a raw buffer."""

    def __init__(self, ptr, count):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": "<f8", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


class Feast:
    """One handle of the C ABI: contour, quadrature, node ownership and workspace."""

    def __init__(self, n, m0, center=0j, r=1.0, aspect=1.0, n_e=8, rule=RULE_TRAPEZOID, mode=RIGHT,
                 b_is_identity=True, rank=0, world=1, max_batch=0, device=None, group=None, real_pencil=False,
                 complex_symmetric=False, segments=None, k_per_segment=8, segment_rule=RULE_TRAPEZOID,
                 partial=False):
        """world > 1 needs an initialised torch.distributed process group of `world` ranks (the
        library then returns node sums over all ranks), or partial=True: every projector call
        returns this rank's partial sum over its own nodes (virtual ranks, caller-side sums)."""
        self.lib = load_library()
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.stream = torch.cuda.current_stream(self.device)
        self.n, self.m0, self.mode, self.b_is_identity = int(n), int(m0), int(mode), bool(b_is_identity)
        self.rank, self.world, self.group = int(rank), int(world), group
        self.center, self.r, self.aspect = complex(center), float(r), float(aspect)
        h = ctypes.c_void_p()
        rc = self.lib.feast_init(ctypes.byref(h), self.n, self.m0, self.center.real, self.center.imag, self.r,
                                 self.aspect, int(n_e), int(rule), self.mode, int(self.b_is_identity), self.rank,
                                 self.world, int(max_batch), ctypes.c_void_p(self.stream.cuda_stream))
        if rc != OK:
            raise FeastError(rc, "feast_init rejected the arguments")
        self.h = h
        if segments is not None:   # composite contour (NEXT-4): [("line", a, b) | ("arc", c, R, th0, th1)]
            kind = (ctypes.c_int32 * len(segments))()
            par = (ctypes.c_double * (5 * len(segments)))()
            for i, sg in enumerate(segments):
                kind[i] = 0 if sg[0] == "line" else 1
                vals = ([complex(sg[1]).real, complex(sg[1]).imag, complex(sg[2]).real, complex(sg[2]).imag, 0.0]
                        if sg[0] == "line" else [complex(sg[1]).real, complex(sg[1]).imag, sg[2], sg[3], sg[4]])
                for k, v in enumerate(vals):
                    par[5 * i + k] = float(v)
            self._check(self.lib.feast_set_contour(self.h, len(segments), kind, par, int(k_per_segment),
                                                   int(segment_rule)))
        self.real_pencil = bool(real_pencil)
        if self.real_pencil:   # conjugate-pole pairs share one LU (NEXT-2b); before the workspace
            self._check(self.lib.feast_set_real_pencil(self.h, 1))
        if complex_symmetric:  # A^T = A, B^T = B: left block through the right solves (NEXT-2a)
            self._check(self.lib.feast_set_complex_symmetric(self.h, 1))
        nbytes = ctypes.c_size_t()
        self._check(self.lib.feast_workspace_bytes(self.h, ctypes.byref(nbytes)))
        self.workspace = torch.empty(int(nbytes.value) + 256, dtype=torch.uint8, device=self.device)
        base = self.workspace.data_ptr()
        aligned = (base + 255) // 256 * 256
        self._check(self.lib.feast_bind_workspace(self.h, ctypes.c_void_p(aligned), int(nbytes.value)))
        self._ar = None
        self.partial = bool(partial)
        if self.world > 1:
            if self.partial:
                self._check(self.lib.feast_set_partial(self.h, 1))
            elif _dist_world(group) == self.world:
                # node sums (and the row-sharded a1 / a7 assemblies) through torch.distributed
                self._ar = ALLREDUCE_FN(make_allreduce_callback(self.device, group))
                self._check(self.lib.feast_set_allreduce(self.h, self._ar, None))
            else:
                self.close()
                raise FeastError(E_COMM, f"world={self.world} needs a torch.distributed process group of that "
                                         f"size (found {_dist_world(group)}) or partial=True")

    # ------------------------------------------------------------------ helpers
    def _check(self, rc, allow_warn=True):
        if rc < 0 or (rc > 0 and not allow_warn):
            raise FeastError(rc, self.lib.feast_last_error(self.h).decode())
        return rc

    def close(self):
        if getattr(self, "h", None):
            self.lib.feast_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    # ------------------------------------------------------------------ API
    def nodes(self):
        q = ctypes.c_int32()
        self._check(self.lib.feast_nodes(self.h, ctypes.byref(q), None, None, None, None))
        z = (ctypes.c_double * (2 * q.value))()
        w = (ctypes.c_double * (2 * q.value))()
        j0, j1 = ctypes.c_int32(), ctypes.c_int32()
        self._check(self.lib.feast_nodes(self.h, None, z, w, ctypes.byref(j0), ctypes.byref(j1)))
        zz = [complex(z[2 * i], z[2 * i + 1]) for i in range(q.value)]
        ww = [complex(w[2 * i], w[2 * i + 1]) for i in range(q.value)]
        return zz, ww, j0.value, j1.value

    def project(self, A, B, X, Q=None):
        """Q = sum_j w_j (z_j B - A)^-1 (B X), node-summed over the ranks by the library
        (partial=True: this rank's nodes only)."""
        Q = empty_colmajor(self.n, self.m0, self.device) if Q is None else Q
        pa, lda = _ptr_ld(A, self.n, "A", self.device, self.n)
        pb, ldb = _ptr_ld(B, self.n, "B", self.device, self.n)
        px, ldx = _ptr_ld(X, self.n, "X", self.device, self.m0)
        pq, ldq = _ptr_ld(Q, self.n, "Q", self.device, self.m0)
        self.status = self._check(self.lib.feast_project(self.h, pa, lda, pb, ldb, px, ldx, pq, ldq))
        return Q

    def project_left(self, A, B, V, QL=None):
        QL = empty_colmajor(self.n, self.m0, self.device) if QL is None else QL
        pa, lda = _ptr_ld(A, self.n, "A", self.device, self.n)
        pb, ldb = _ptr_ld(B, self.n, "B", self.device, self.n)
        pv, ldv = _ptr_ld(V, self.n, "V", self.device, self.m0)
        pq, ldq = _ptr_ld(QL, self.n, "QL", self.device, self.m0)
        self.status = self._check(self.lib.feast_project_left(self.h, pa, lda, pb, ldb, pv, ldv, pq, ldq))
        return QL

    def project_bi(self, A, B, X, V, Q=None, QL=None):
        Q = empty_colmajor(self.n, self.m0, self.device) if Q is None else Q
        QL = empty_colmajor(self.n, self.m0, self.device) if QL is None else QL
        pa, lda = _ptr_ld(A, self.n, "A", self.device, self.n)
        pb, ldb = _ptr_ld(B, self.n, "B", self.device, self.n)
        px, ldx = _ptr_ld(X, self.n, "X", self.device, self.m0)
        pv, ldv = _ptr_ld(V, self.n, "V", self.device, self.m0)
        pq, ldq = _ptr_ld(Q, self.n, "Q", self.device, self.m0)
        pl, ldl = _ptr_ld(QL, self.n, "QL", self.device, self.m0)
        self.status = self._check(self.lib.feast_project_bi(self.h, pa, lda, pb, ldb, px, ldx, pv, ldv, pq, ldq,
                                                            pl, ldl))
        return Q, QL

    def reduce(self, A, B, Q, QL=None, Ahat=None, Bhat=None):
        Ahat = empty_colmajor(self.m0, self.m0, self.device) if Ahat is None else Ahat
        Bhat = empty_colmajor(self.m0, self.m0, self.device) if Bhat is None else Bhat
        pa, lda = _ptr_ld(A, self.n, "A", self.device, self.n)
        pb, ldb = _ptr_ld(B, self.n, "B", self.device, self.n)
        pq, ldq = _ptr_ld(Q, self.n, "Q", self.device, self.m0)
        pl, ldl = _ptr_ld(QL, self.n, "QL", self.device, self.m0)
        p1, ld1 = _ptr_ld(Ahat, self.m0, "Ahat", self.device, self.m0)
        p2, ld2 = _ptr_ld(Bhat, self.m0, "Bhat", self.device, self.m0)
        self._check(self.lib.feast_reduce(self.h, pa, lda, pb, ldb, pq, ldq, pl, ldl, p1, ld1, p2, ld2))
        return Ahat, Bhat

    def iterate(self, A, B, X, V=None):
        """One R-FEAST / Bi-FEAST iteration; X (and V) updated in place."""
        m = self.m0
        ritz = (ctypes.c_double * (2 * m))()
        res = (ctypes.c_double * m)()
        flags = (ctypes.c_int32 * m)()
        pa, lda = _ptr_ld(A, self.n, "A", self.device, self.n)
        pb, ldb = _ptr_ld(B, self.n, "B", self.device, self.n)
        px, ldx = _ptr_ld(X, self.n, "X", self.device, self.m0)
        pv, ldv = _ptr_ld(V, self.n, "V", self.device, self.m0)
        self.status = self._check(self.lib.feast_iterate(self.h, pa, lda, pb, ldb, px, ldx, pv, ldv, ritz, res,
                                                         flags))
        lam = [complex(ritz[2 * i], ritz[2 * i + 1]) for i in range(m)]
        return {"lam": lam, "resid": list(res), "flags": list(flags)}

    def filter(self, mu):
        """rho(mu) = sum_j w_j / (z_j - mu) of this handle's quadrature at host points mu."""
        import numpy as np
        mu = np.ascontiguousarray(np.atleast_1d(mu), dtype=np.complex128)
        out = np.zeros_like(mu)
        self._check(self.lib.feast_filter(self.h, len(mu), mu.ctypes.data_as(ctypes.c_void_p),
                                          out.ctypes.data_as(ctypes.c_void_p)))
        return out

    def estimate_count(self, A, B, U, Q=None):
        """Eigenvalue-count estimate Re tr(U^H rho(B^-1 A) U) / m0 for a random block U (NEXT-3);
        returns (estimate, Q = rho(B^-1 A) U, node-summed over ranks)."""
        Q = empty_colmajor(self.n, self.m0, self.device) if Q is None else Q
        pa, lda = _ptr_ld(A, self.n, "A", self.device, self.n)
        pb, ldb = _ptr_ld(B, self.n, "B", self.device, self.n)
        pu, ldu = _ptr_ld(U, self.n, "U", self.device, self.m0)
        pq, ldq = _ptr_ld(Q, self.n, "Q", self.device, self.m0)
        est = ctypes.c_double()
        self.status = self._check(self.lib.feast_estimate_count(self.h, pa, lda, pb, ldb, pu, ldu, pq, ldq,
                                                                ctypes.byref(est)))
        return est.value, Q

    def estimate_count_bi(self, A, B, U, V, Q=None, QL=None):
        """Count estimate from eig(V^^H B U^) of Bi-FEAST steps 4-5 (reading R21):
        returns (count, mu sorted by decreasing modulus, Q = U^, QL = V^)."""
        import numpy as np
        Q = empty_colmajor(self.n, self.m0, self.device) if Q is None else Q
        QL = empty_colmajor(self.n, self.m0, self.device) if QL is None else QL
        pa, lda = _ptr_ld(A, self.n, "A", self.device, self.n)
        pb, ldb = _ptr_ld(B, self.n, "B", self.device, self.n)
        pu, ldu = _ptr_ld(U, self.n, "U", self.device, self.m0)
        pv, ldv = _ptr_ld(V, self.n, "V", self.device, self.m0)
        pq, ldq = _ptr_ld(Q, self.n, "Q", self.device, self.m0)
        pl, ldl = _ptr_ld(QL, self.n, "QL", self.device, self.m0)
        mu = np.zeros(self.m0, dtype=np.complex128)
        cnt = ctypes.c_int32()
        self.status = self._check(self.lib.feast_estimate_count_bi(
            self.h, pa, lda, pb, ldb, pu, ldu, pv, ldv, pq, ldq, pl, ldl, mu.ctypes.data_as(ctypes.c_void_p),
            ctypes.byref(cnt)))
        return cnt.value, mu, Q, QL

    def set_async(self, enable: bool):
        """Projector / reduce calls return once enqueued (no host synchronisation); sync() waits
        and returns the last projection's status (raises on FEAST_E_SINGULAR)."""
        self._check(self.lib.feast_set_async(self.h, int(bool(enable))))

    def sync(self):
        self.status = self._check(self.lib.feast_sync(self.h))
        return self.status

    def set_count_estimate(self, enable: bool):
        """Track the eig(V^^H B U^) count estimate in every Bi-FEAST iterate() (see monitors())."""
        self._check(self.lib.feast_set_count_estimate(self.h, int(bool(enable))))

    def monitors(self):
        """Res_(k), trace_(k), number of candidates of the last iterate(), and (Bi-FEAST
        with set_count_estimate) the count estimate and eig(V^^H B U^) sorted by modulus."""
        import numpy as np
        res, tr, nc, cnt = ctypes.c_double(), (ctypes.c_double * 2)(), ctypes.c_int32(), ctypes.c_int32()
        mu = np.zeros(self.m0, dtype=np.complex128)
        self._check(self.lib.feast_monitors(self.h, ctypes.byref(res), tr, ctypes.byref(nc),
                                            mu.ctypes.data_as(ctypes.c_void_p), ctypes.byref(cnt)))
        return {"res_k": res.value, "trace_k": complex(tr[0], tr[1]), "ncand": nc.value, "count": cnt.value,
                "mu": mu if cnt.value >= 0 else None}

    def filter_gap(self, lam, p):
        """Filter-gap report of eigenvalues lam (host) for subspace size p."""
        import numpy as np
        lam = np.ascontiguousarray(np.atleast_1d(lam), dtype=np.complex128)
        nl = len(lam)
        a = np.zeros(nl)
        order = np.zeros(nl, dtype=np.int32)
        m, mp, eps, lg = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_double(), ctypes.c_double()
        self._check(self.lib.feast_filter_gap(self.h, nl, lam.ctypes.data_as(ctypes.c_void_p), int(p),
                                              a.ctypes.data_as(ctypes.c_void_p), order.ctypes.data_as(ctypes.c_void_p),
                                              ctypes.byref(m), ctypes.byref(mp), ctypes.byref(eps), ctypes.byref(lg)))
        return dict(abs_sorted=a, order=order.astype(np.int64), m=m.value, m_prime=mp.value, eps=eps.value,
                    log10_gap=lg.value)

    def node_stats(self):
        zz, _, _, _ = self.nodes()
        arr = (ctypes.c_double * len(zz))()
        worst = ctypes.c_int32()
        self._check(self.lib.feast_node_stats(self.h, arr, ctypes.byref(worst)))
        return list(arr), worst.value

    def factor_cache(self, enable: bool):
        """Factor-once reuse across calls with the same A, B (NEXT-1); enable=True invalidates."""
        self._check(self.lib.feast_factor_cache(self.h, int(bool(enable))))

    def profile(self, enable, serial: bool = False):
        """Start (clears) / stop per-kernel-class CUDA-event timing of this library's launches;
        serial=True serialises every launch on one stream so each event pair times one kernel."""
        self._check(self.lib.feast_profile(self.h, (2 if serial else 1) if enable else 0))

    def profile_summary(self):
        """{class: {launches, ms, flops, bytes}} of the launches recorded since profile(True)."""
        out = {}
        for i, name in enumerate(K_CLASSES):
            c, ms, fl, by = ctypes.c_int64(), ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
            self._check(self.lib.feast_profile_summary(self.h, i, ctypes.byref(c), ctypes.byref(ms), ctypes.byref(fl),
                                                       ctypes.byref(by)))
            out[name] = {"launches": c.value, "ms": ms.value, "flops": fl.value, "bytes": by.value}
        return out

    def profile_records(self, max_records: int = 100000):
        """Per-launch timeline since profile(True): list of (class, stream, t0_ms, t1_ms, flops)."""
        cnt = ctypes.c_int64()
        self._check(self.lib.feast_profile_records(self.h, 0, None, None, None, None, None, ctypes.byref(cnt)))
        m = min(cnt.value, max_records)
        cl, st = (ctypes.c_int32 * m)(), (ctypes.c_int32 * m)()
        t0, t1, fl = (ctypes.c_double * m)(), (ctypes.c_double * m)(), (ctypes.c_double * m)()
        self._check(self.lib.feast_profile_records(self.h, m, cl, st, t0, t1, fl, ctypes.byref(cnt)))
        return [(K_CLASSES[cl[i]], st[i], t0[i], t1[i], fl[i]) for i in range(m)]

    @property
    def last_launch_count(self) -> int:
        return int(self.lib.feast_last_launch_count(self.h))
