"""bench.py — FEAST quadrature-projector hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl reference]

A STEP is one pass of the whole hot path over the synthetic pencil of
the chosen config, through the C ABI:
  a1 R = B X (B^H V), a2 C_j = z_j B - A, a3 P_j C_j = L_j U_j, a4 Y_j = C_j^-1 R (Bi-FEAST: and
  Z_j = C_j^-H R_L from the same factors), a5 Q = sum w_j Y_j (QL = sum conj(w_j) Z_j) over all q
  nodes sharded over the ranks, a6 the node sum over ranks (inside the library, through the
  registered torch.distributed callback: NCCL), a7 Ahat = QL^H A Q, Bhat = QL^H B Q (rows sharded).
The m0 x m0 reduced eigenproblem lies outside the timed hot path (BASELINE north_star).

Default workload C4 (BASELINE.json configs[3]: n = 16384, m0 = 512, q = 32, Bi-FEAST), the
largest config that fits one GPU (BASELINE's metric names no config; C5 is quoted "2 per GPU on
8 x B200").  `value` = FEAST iterations per second of the whole job (strong scaling: the problem
is fixed and its q nodes are split over the N ranks).

Timing: W untimed warm-up steps; K timed steps bracketed by barrier + cuda.synchronize on both
sides; CUDA events on the library's stream; max over ranks.  Every C4 step streams the 32
augmented LU workspaces (~140 GB) through HBM, far more than the 126 MB L2 (no flush needed).

--gpus N without an outer torchrun re-launches this script under torch.distributed.run with N
ranks (one per GPU).  --impl reference runs the plain-C oracle (oracle/) on the host cores
instead: the reference arm of this tier (a deliberately slow program, timed on a bounded
sample and extrapolated by flops; parity and roofline are the headline).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FEAST iterations/sec and shifted LU+solve FP64 TFLOP/s (% peak) at 1/2/4/8 GPUs"
FP64_PEAK_TFLOPS = 37.17     # measured DMMA peak, profiles/r01_fp64_peak.md (MEASURED_PEAKS.json has no FP64)
FP64_PEAK_NOTE = ("measured DMMA.8x8x4 throughput on this pool's B200 (tools/fp64_peak.cu, profiles/r01_fp64_peak.md; "
                  "MEASURED_PEAKS.json has no FP64 entry); datasheet 37.2 at 1965 MHz")
DEFAULT_CONFIG = "C4"


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:  # noqa: BLE001
        return {}


def _flops(spec, n, m0, q):
    """Algorithmic flops of one step: LU + solves per node, B X (B^H V), A Q (+ B Q),
    QL^H (.).  Returns (shifted LU + solve flops, total)."""
    bi = 2 if spec.mode == "bi" else 1
    bnot = 0 if spec.b_is_identity else 1
    lu_solve = q * (8.0 / 3.0 * n ** 3 + 8.0 * n * n * m0 * bi)
    total = lu_solve + bnot * 8.0 * n * n * m0 * bi + 8.0 * n * n * m0 * (1 + bnot) + 2 * 8.0 * n * m0 * m0
    return lu_solve, total


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:  # noqa: BLE001
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        rows = [r.split(",") for r in open(self.path).read().strip().splitlines() if r.strip()]
        os.unlink(self.path)
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].strip().replace(".", "").isdigit()]
        smax = [float(r[2]) for r in rows if len(r) >= 9 and r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            if len(r) < 9:
                continue
            for name, v in zip(names, r[5:9]):
                if v.strip() == "Active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(rows)}


def _dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _relaunch(args):
    """--gpus N > 1 without an outer launcher: run this script under torch.distributed.run, one
    rank per GPU, and return its exit code (rank 0 prints the JSON line)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__),
           *sys.argv[1:]]
    return subprocess.call(cmd)


# ------------------------------------------------------------------ the oracle on the host
def _oracle_sample(config, n_s):
    """One bounded sample of the workload on the oracle (plain C, OpenMP over nodes): the
    config's recipe at n_s <= n (m0 scaled by n_s/n), its projector(s) on k = min(q, cores)
    nodes in parallel (one per core; Bi-FEAST: right and left), plus the oracle reduce
    (A Q, QL^H A Q, QL^H B Q).  Returns (seconds, algorithmic flops of the sample, description)."""
    import numpy as np

    import oracle
    import synth
    spec = synth.CONFIGS[config]
    n_s = min(spec.n, n_s)
    m_s = max(1, spec.m0 * n_s // spec.n)
    P = synth.make_pencil(config, n=n_s, m0=m_s)
    z, w = oracle.nodes(spec.c, spec.r, spec.aspect, spec.n_e, spec.rule)
    cores = oracle.threads(len(os.sched_getaffinity(0)))   # every host core (torchrun sets OMP_NUM_THREADS=1)
    q = len(z)
    k = min(q, cores)
    bi = spec.mode == "bi"
    V0 = P.X0 @ np.linalg.inv(P.X0.conj().T @ P.X0).conj().T if bi else None   # reading R6 (fixture)
    t0 = time.perf_counter()
    Q = oracle.project(P.A, P.B, P.X0, z, w, 0, k)
    QL = oracle.project(P.A, P.B, V0, z, w, 0, k, left=True) if bi else Q
    AQ = oracle.gemm(P.A, Q)
    oracle.gemm(QL, AQ, opa=2)
    oracle.gemm(QL, Q if P.B is None else oracle.gemm(P.B, Q), opa=2)
    sec = time.perf_counter() - t0
    lu_solve, _ = _flops(spec, n_s, m_s, k)
    _, total_1 = _flops(spec, n_s, m_s, 0)        # the reduce (and B X) part at the sample size
    desc = (f"{config} recipe at n={n_s}, m0={m_s}: oracle projector{'s (right+left)' if bi else ''} on {k} of {q} "
            f"nodes in parallel (one per core) + oracle reduce; {sec:.1f} s; extrapolated to n={spec.n}, "
            f"m0={spec.m0}, q={q} by algorithmic flops at the sample's rate (the naive LU only slows down further "
            f"at full size, so this overstates the oracle)")
    return sec, lu_solve + total_1, desc, min(k, cores)


def cpu_baseline(config, n_s=2048):
    import synth
    spec = synth.CONFIGS[config]
    sec, fl, desc, cores = _oracle_sample(config, n_s)
    _, full = _flops(spec, spec.n, spec.m0, spec.q)
    full_sec = full / (fl / sec)
    return {"value": 1.0 / full_sec, "unit": "iter/s", "cores": cores, "kind": "oracle", "sample": desc,
            "extrapolated": True, "sample_gflops": fl / sec / 1e9}


def run_reference(args):
    """Reference arm: the oracle (plain C, OpenMP over nodes) on this host's cores, each step a
    bounded sample of the workload extrapolated by flops (rank 0 only)."""
    import synth
    rank, world, _ = _dist_env()
    if rank != 0:
        return 0
    spec = synth.CONFIGS[args.config]
    _, full = _flops(spec, spec.n, spec.m0, spec.q)
    lu_solve, _ = _flops(spec, spec.n, spec.m0, spec.q)
    n_s = 1024
    for _ in range(args.warmup):
        _oracle_sample(args.config, n_s)
    secs, desc, cores = [], "", 0
    for _ in range(args.steps):
        sec, fl, desc, cores = _oracle_sample(args.config, n_s)
        secs.append(full / (fl / sec))
    ms = 1e3 * sum(secs) / len(secs)
    value = 1e3 / ms
    line = {"metric": METRIC, "value": value, "unit": "iter/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "complex128", "data": "synthetic", "impl": "reference",
            "config": {"workload": args.config, "n": spec.n, "m0": spec.m0, "q": spec.q, "mode": spec.mode},
            "lu_solve_tflops": lu_solve / (ms * 1e-3) / 1e12,
            "cpu_baseline": {"value": value, "unit": "iter/s", "cores": cores, "kind": "oracle",
                             "sample": "every step: " + desc, "extrapolated": True},
            "e2e": {"value": value, "unit": "iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ launcher dry run (CPU)
def run_dry(args):
    """Launcher / rank plumbing only (no GPU, no hot path): gloo process group, barrier, a
    per-rank dummy time reduced with MAX, rank 0 prints n_gpus — tested on CPU."""
    import torch
    import torch.distributed as dist
    rank, world, _ = _dist_env()
    if world != args.gpus:
        print(f"bench: WORLD_SIZE={world} != --gpus {args.gpus}", file=sys.stderr)
        return 2
    if world > 1:
        dist.init_process_group("gloo")
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "max_rank_time": float(t.item()), "config": args.config}),
              flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


# ------------------------------------------------------------------ the GPU arm
def run_gpu(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import synth
    from paper_1404_2891_b200 import Feast, empty_colmajor, feast as fb

    rank, world, local = _dist_env()
    if world != args.gpus:
        print(f"bench: WORLD_SIZE={world} != --gpus {args.gpus}", file=sys.stderr)
        return 2
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    spec = synth.CONFIGS[args.config]
    bi = spec.mode == "bi"
    # fixture (seeded, synthetic; A built with a library solve — not the method)
    P = synth.make_pencil_torch(args.config) if spec.n >= 4096 else None
    if P is None:
        Ph = synth.make_pencil(args.config)
        dev = lambda a: None if a is None else torch.from_numpy(np.asfortranarray(a)).to("cuda")
        A, B, X = dev(Ph.A), dev(Ph.B), dev(Ph.X0)
        n, m0, q = Ph.n, Ph.m0, Ph.q
    else:
        A, B, X = P.A, P.B, P.X0
        n, m0, q = P.n, P.m0, P.q
        P.V = None   # the spectral data is for parity tests, not the bench
        P.lam = None
    V = None
    if bi:   # V^(0) = X0 G^-H, G = X0^H B X0 (reading R6; B = I in C4)
        G = X.conj().T @ (X if B is None else B @ X)
        V = fb.colmajor(torch.linalg.solve(G, X.conj().T).conj().T)
        del G
    del P
    torch.cuda.empty_cache()
    f = Feast(n, m0, spec.c, spec.r, spec.aspect, spec.n_e, spec.rule, fb.BI if bi else fb.RIGHT, B is None,
              rank=rank, world=world)
    f.set_async(True)      # steps pipeline on the stream; the status is checked by f.sync()
    stream = f.stream
    Q = empty_colmajor(n, m0)
    QL = empty_colmajor(n, m0) if bi else None
    Ah = empty_colmajor(m0, m0)
    Bh = empty_colmajor(m0, m0)
    launches = [0]

    def step():
        if bi:
            f.project_bi(A, B, X, V, Q, QL)   # a1-a6 (node sum over ranks inside the library)
        else:
            f.project(A, B, X, Q)
        c = f.last_launch_count
        f.reduce(A, B, Q, QL, Ah, Bh)         # a7, rows sharded over ranks
        launches[0] = c + f.last_launch_count

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if world > 1:
            t = torch.tensor([v], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            v = float(t.item())
        return v

    for _ in range(max(args.warmup, 0)):
        step()
    barrier()
    clk = ClockSampler(local)
    clk.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    barrier()
    clocks = clk.stop()
    f.sync()               # raises if a node's shifted matrix was singular
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    gpu_launches = launches[0] * args.steps
    bounded = max(1, min(2, args.steps)) if ms > 2000 else max(1, min(3, args.steps))
    if args.timing_only:   # experiments (A/B of knobs): the timed steps alone, no extra passes
        if rank == 0:
            lu_solve, total = _flops(spec, n, m0, q)
            print(json.dumps({"timing_only": True, "config": args.config, "n_gpus": world, "ms_per_step": ms,
                              "value": 1e3 / ms, "lu_solve_frac_peak": lu_solve / (ms * 1e-3) / 1e12 /
                              FP64_PEAK_TFLOPS / world, "clocks": clocks, "gpu_launches": gpu_launches,
                              "env": {k: v for k, v in os.environ.items() if k.startswith("FEAST_")}}), flush=True)
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    # ---- per-kernel-class timing: CUDA events around every launch on its launching stream, in a
    # SERIALISED pass after the timed region (one stream, no lookahead / node groups / graph), so
    # each event pair brackets exactly one kernel; the timed region itself runs the overlapped
    # schedule (graph replay, concurrent node groups), where a kernel's events would also count
    # time spent queued behind other streams' kernels.
    f.profile(True, serial=True)
    prof_steps = 1
    for _ in range(prof_steps):
        step()
    torch.cuda.synchronize()
    prof = f.profile_summary()
    f.profile(False)
    zg = prof["zgemm"]
    achieved = zg["flops"] / (zg["ms"] * 1e-3) / 1e12 if zg["ms"] > 0 else 0.0
    total_prof_ms = sum(v["ms"] for v in prof.values())
    traffic, traffic_src = None, None
    traffic_ratio = None
    try:  # committed ncu capture of the same serialised step (tools/zgemm_traffic.py)
        tp = os.path.join("profiles", f"zgemm_traffic_{args.config}.json")
        tr = json.load(open(os.path.join(ROOT, tp)))
        if tr.get("config") == args.config:
            traffic_ratio = tr.get("traffic_over_algorithmic")
            # DRAM bytes per launch: the captured ratio to the algorithmic bytes applied to this
            # run's launches (the same kernels; the capture's own per-launch mean is in the file)
            traffic = traffic_ratio * zg["bytes"] / max(1, zg["launches"]) if traffic_ratio else None
            traffic_src = f"{tp} (ncu dram__bytes_read+write of every zgemm launch of one serialised step, " \
                          f"{tr.get('launches')} launches: {traffic_ratio:.3f} x algorithmic bytes)"
    except Exception:  # noqa: BLE001
        pass
    hbm = _peaks().get("hbm_gbs")
    per_class_gbs = {k: (v["bytes"] / (v["ms"] * 1e-3) / 1e9 if v["ms"] > 0 else None)
                     for k, v in prof.items() if k in ("shift", "laswp", "perm", "accum")}
    roofline = {"bound": "tensor", "kernel": "zgemm_dmma_kernel (FP64 DMMA.8x8x4)", "achieved": achieved,
                "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS,
                "traffic": traffic, "traffic_over_algorithmic": traffic_ratio, "peak_source": FP64_PEAK_NOTE,
                "launches_per_step": zg["launches"] / prof_steps,
                "algorithmic_flops_per_launch": zg["flops"] / max(1, zg["launches"]),
                "algorithmic_bytes_per_launch": zg["bytes"] / max(1, zg["launches"]),
                "flops_convention": "8 M N K per complex GEMM; 4 K (K+1) N for the in-place 64x64 triangular-inverse "
                                    "products (the executed dense 8 K^2 N is not counted)",
                "traffic_source": traffic_src,
                "share_of_serialised_step": zg["ms"] / total_prof_ms if total_prof_ms > 0 else None,
                "serialised_step_ms": total_prof_ms / prof_steps,
                "timing": "CUDA events per launch on its stream, serialised pass after the timed region",
                "per_class_ms_per_step": {k: v["ms"] / prof_steps for k, v in prof.items()},
                "per_class_launches_per_step": {k: v["launches"] / prof_steps for k, v in prof.items()},
                "hbm_kernels_gbs": per_class_gbs,
                "hbm_kernels_note": "laswp counts only the rows that actually move (device counter): the BASELINE "
                                    "pencils pivot (almost) on the diagonal, so it moves ~nothing; the swap kernels' "
                                    "bandwidth on a pivot-heavy pencil is in profiles/r02/swap_ncu.txt",
                "hbm_peak_gbs": hbm, "hbm_peak_source": "MEASURED_PEAKS.json hbm_gbs (driver-measured copy bandwidth)"}

    # ---- end to end through the public API with pinned host buffers: every step copies the
    # step's inputs (A, B, X, V) host -> device and reads the reduced matrices back
    def pin(t):   # pinned host copy with the device tensor's (column-major) strides: one flat memcpy
        if t is None:
            return None
        h = torch.empty_strided(t.shape, t.stride(), dtype=t.dtype, pin_memory=True)
        h.copy_(t)
        return h

    pinA, pinB, pinX, pinV = pin(A), pin(B), pin(X), pin(V)
    outA = torch.empty((m0, m0), dtype=torch.complex128).pin_memory().t()
    outB = torch.empty((m0, m0), dtype=torch.complex128).pin_memory().t()
    h2d = sum(t.numel() * 16 for t in (pinA, pinB, pinX, pinV) if t is not None)
    d2h = 2 * m0 * m0 * 16

    def e2e_step():
        for d, h in ((A, pinA), (B, pinB), (X, pinX), (V, pinV)):
            if h is not None:
                d.copy_(h, non_blocking=True)
        step()
        outA.copy_(Ah, non_blocking=True)
        outB.copy_(Bh, non_blocking=True)

    e2e_step()
    barrier()
    e0.record(stream)
    for _ in range(bounded):
        e2e_step()
    e1.record(stream)
    barrier()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1) / bounded)

    # ---- full FEAST iterations (SURVEY §8(d) metric (1) "including the reduced eig"): projector,
    # node sum, orthonormalisation, reduced matrices, reduced eigenproblem (cuSOLVER), Ritz
    # vectors and residuals — feast_iterate through the public API, inputs resident.
    Xit, Vit = X.clone(), (V.clone() if bi else None)
    f.iterate(A, B, Xit, Vit)
    barrier()
    e0.record(f.stream)
    n_it = 1 if ms > 2000 else 3
    for _ in range(n_it):
        f.iterate(A, B, Xit, Vit)
    e1.record(f.stream)
    barrier()
    it_ms = max_over_ranks(e0.elapsed_time(e1) / n_it)

    lu_solve, total = _flops(spec, n, m0, q)
    if rank == 0:
        bdesc = "I" if B is None else f"I + {spec.bscale} G_B/sqrt(n)"
        line = {"metric": METRIC, "value": 1e3 / ms, "unit": "iter/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "complex128", "data": "synthetic",
                "config": {"workload": args.config, "n": n, "m0": m0, "q": q,
                           "rule": {0: "trapezoid(midpoint)", 1: "trapezoid(endpoint)", 2: "gauss-legendre"}[spec.rule],
                           "B": bdesc, "mode": spec.mode, "parallelism": f"nodes{world}", "nodes_per_rank": q // world,
                           "l2": "no flush: every step streams the q augmented LU workspaces (16 n (n + m0) bytes "
                                 "each) through HBM, far larger than the 126 MB L2"},
                "lu_solve_tflops": lu_solve / (ms * 1e-3) / 1e12,
                "lu_solve_frac_peak": lu_solve / (ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS / world,
                "step_tflops": total / (ms * 1e-3) / 1e12,
                "step_frac_peak": total / (ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS / world,
                "clocks": clocks, "gpu_launches": gpu_launches,
                "e2e": {"value": 1e3 / e2e_ms, "unit": "iter/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                        "steps": bounded},
                "iteration_incl_reduced_eig": {"value": 1e3 / it_ms, "unit": "iter/s", "ms": it_ms,
                                               "what": "feast_iterate: projector(s) + node sum + QR + reduced "
                                                       "matrices + reduced eig (cuSOLVER Xgeev) + Ritz vectors/"
                                                       "residuals"},
                "roofline": roofline}
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(args.config)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=DEFAULT_CONFIG)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dry-run", action="store_true", help="launcher / rank plumbing only (CPU, gloo)")
    ap.add_argument("--timing-only", action="store_true", help="experiments: the timed steps only (no profile, "
                                                               "e2e, iterate or oracle passes)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return _relaunch(args)
    if args.dry_run:
        return run_dry(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
