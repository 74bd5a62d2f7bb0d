"""bench.py — FEAST quadrature-projector hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl reference]

A STEP is one pass of the whole hot path over the synthetic pencil
of config C2 (BASELINE.json configs[1], the config the metric is quoted on; it fits one GPU):
  a1 R = B X, a2 C_j = z_j B - A, a3 P_j C_j = L_j U_j, a4 Y_j = C_j^-1 R, a5 Q = sum w_j Y_j
  (all q nodes, sharded over ranks), a6 all-reduce of Q (N > 1), a7 Ahat = Q^H A Q, Bhat = Q^H B Q.
The m0 x m0 reduced eigenproblem lies outside the timed hot path (BASELINE north_star).
`value` = FEAST iterations per second of the whole job (strong scaling: the problem is fixed
and its q nodes are split over the N ranks).

Timing: W untimed warm-up steps; K timed steps bracketed by barrier + cuda.synchronize on both
sides; CUDA events on the library's stream; max over ranks.  Every step streams > 1 GB
(the q LU workspaces) through HBM, larger than the 126 MB L2.

--impl reference runs the plain-C oracle (oracle/) on the host cores instead: the reference
arm of this tier (a deliberately slow program; parity and roofline are the headline).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FEAST iterations/sec and shifted LU+solve FP64 TFLOP/s (% peak) at 1/2/4/8 GPUs"
FP64_PEAK_TFLOPS = 37.17     # measured DMMA peak, profiles/r01_fp64_peak.md (MEASURED_PEAKS.json has no FP64)
FP64_PEAK_NOTE = "measured DMMA.8x8x4 peak on this pool's B200 (profiles/r01_fp64_peak.md); datasheet 37.2"


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:  # noqa: BLE001
        return {}


def _flops(spec, n, m0, q):
    """Algorithmic flops of one step: LU + solves per node, B X, A Q (+ B Q), Q^H(.)."""
    bi = spec.mode == "bi"
    bnot = 0 if spec.b_is_identity else 1
    lu_solve = q * (8.0 / 3.0 * n ** 3 + 8.0 * n * n * m0 * (2 if bi else 1))
    total = lu_solve + bnot * 8.0 * n * n * m0 * (2 if bi else 1) + 8.0 * n * n * m0 * (1 + bnot) + 2 * 8.0 * n * m0 * m0
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
                                          "--format=csv,noheader,nounits", "-lms", "100"],
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


def run_reference(args):
    """Reference arm: the oracle (plain C, OpenMP over nodes) on this host's cores."""
    import numpy as np

    import oracle
    import synth
    rank, world, _ = _dist_env()
    if rank != 0:
        return 0
    spec = synth.CONFIGS[args.config]
    P = synth.make_pencil(args.config)
    z, w = oracle.nodes(spec.c, spec.r, spec.aspect, spec.n_e, spec.rule)
    cores = len(os.sched_getaffinity(0))
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    q = len(z)
    nodes = min(q, cores)                     # one node per core: a bounded sample of the step
    lu_solve, total = _flops(spec, P.n, P.m0, q)

    def step():
        t0 = time.perf_counter()
        oracle.project(P.A, P.B, P.X0, z, w, 0, nodes)
        t1 = time.perf_counter()
        Q = P.X0
        AQ = oracle.gemm(P.A, Q)
        oracle.gemm(Q, AQ, opa=2)
        if P.B is not None:
            oracle.gemm(Q, oracle.gemm(P.B, Q), opa=2)
        t2 = time.perf_counter()
        return (t1 - t0) * (q / nodes) + (t2 - t1)   # extrapolated to all q nodes

    for _ in range(args.warmup):
        step()
    times = [step() for _ in range(args.steps)]
    ms = 1e3 * sum(times) / len(times)
    value = 1e3 / ms
    sample = (f"{args.config}: oracle projector on {nodes} of {q} nodes (one per core, in parallel), scaled by "
              f"q/{nodes}, plus the oracle reduce (A Q, Q^H A Q, Q^H B Q) in full")
    line = {"metric": METRIC, "value": value, "unit": "iter/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "complex128", "data": "synthetic", "impl": "reference",
            "config": {"workload": args.config, "n": P.n, "m0": P.m0, "q": q},
            "lu_solve_tflops": lu_solve / (ms * 1e-3) / 1e12,
            "cpu_baseline": {"value": value, "unit": "iter/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline(args, P, z, w):
    """The oracle, as it stands, on a bounded sample: one step of the same workload with the
    projector limited to min(q, cores) nodes run in parallel (one per core), scaled to q."""
    import oracle
    cores = len(os.sched_getaffinity(0))
    q = len(z)
    nodes = min(q, cores)
    t0 = time.perf_counter()
    oracle.project(P.A, P.B, P.X0, z, w, 0, nodes)
    t1 = time.perf_counter()
    AQ = oracle.gemm(P.A, P.X0)
    oracle.gemm(P.X0, AQ, opa=2)
    if P.B is not None:
        oracle.gemm(P.X0, oracle.gemm(P.B, P.X0), opa=2)
    t2 = time.perf_counter()
    sec = (t1 - t0) * (q / nodes) + (t2 - t1)
    return {"value": 1.0 / sec, "unit": "iter/s", "cores": cores, "kind": "oracle",
            "sample": f"one {args.config} step: oracle projector on {nodes} of {q} nodes in parallel "
                      f"(x q/{nodes}) + full oracle reduce; {t2 - t0:.1f} s of CPU wall time"}


def run_gpu(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import synth
    from paper_1404_2891_b200 import Feast, empty_colmajor, feast as fb

    rank, world, local = _dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    spec = synth.CONFIGS[args.config]
    P = synth.make_pencil(args.config)
    n, m0 = P.n, P.m0
    f = Feast(n, m0, spec.c, spec.r, spec.aspect, spec.n_e, spec.rule, fb.RIGHT, P.B is None, rank=rank, world=world)
    q = P.q
    stream = f.stream
    dev = lambda a: None if a is None else torch.from_numpy(np.asfortranarray(a)).to("cuda")
    A, B, X = dev(P.A), dev(P.B), dev(P.X0)
    Q = empty_colmajor(n, m0)
    Ah = empty_colmajor(m0, m0)
    Bh = empty_colmajor(m0, m0)

    launches = [0]

    def step():
        f.project(A, B, X, Q, allreduce=False)
        c = f.last_launch_count
        f.allreduce_(Q)                                  # a6: node sum over ranks (NCCL)
        f.reduce(A, B, Q, None, Ah, Bh)                  # a7
        launches[0] = c + f.last_launch_count

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

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
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    gpu_launches = launches[0] * args.steps

    # ---- per-kernel-class timing: CUDA events around every launch on its launching stream, in a
    # SERIALISED pass right after the timed region (one stream, no lookahead / node groups /
    # graph), so each event pair brackets exactly one kernel; the timed region itself runs the
    # overlapped schedule (graph replay, concurrent node groups), where a kernel's events would
    # also count time spent queued behind the other stream's kernels.
    f.profile(True, serial=True)
    prof_steps = max(1, min(3, args.steps))
    for _ in range(prof_steps):
        step()
    torch.cuda.synchronize()
    prof = f.profile_summary()
    f.profile(False)
    zg = prof["zgemm"]
    achieved = zg["flops"] / (zg["ms"] * 1e-3) / 1e12 if zg["ms"] > 0 else 0.0
    total_prof_ms = sum(v["ms"] for v in prof.values())
    traffic, traffic_src = None, None
    try:  # committed ncu capture of the same serialised step (tools/zgemm_traffic.py)
        tr = json.load(open(os.path.join(ROOT, "profiles", "zgemm_traffic.json")))
        if tr.get("config") == args.config:
            traffic = tr.get("dram_bytes_per_launch")
            traffic_src = "profiles/zgemm_traffic.json: " + tr.get("source", "")
    except Exception:  # noqa: BLE001
        pass
    roofline = {"bound": "tensor", "kernel": "zgemm_dmma_kernel (FP64 DMMA.8x8x4)", "achieved": achieved,
                "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS,
                "traffic": traffic, "peak_source": FP64_PEAK_NOTE,
                "launches_per_step": zg["launches"] / prof_steps,
                "algorithmic_flops_per_launch": zg["flops"] / max(1, zg["launches"]),
                "algorithmic_bytes_per_launch": zg["bytes"] / max(1, zg["launches"]),
                "traffic_source": traffic_src,
                "share_of_serialised_step": zg["ms"] / total_prof_ms if total_prof_ms > 0 else None,
                "serialised_step_ms": total_prof_ms / prof_steps,
                "timing": "CUDA events per launch on its stream, serialised pass after the timed region",
                "per_class_ms_per_step": {k: v["ms"] / prof_steps for k, v in prof.items()},
                "per_class_launches_per_step": {k: v["launches"] / prof_steps for k, v in prof.items()}}

    # ---- end to end through the public API with pinned host buffers
    pinA = torch.from_numpy(np.asfortranarray(P.A)).pin_memory()
    pinB = None if P.B is None else torch.from_numpy(np.asfortranarray(P.B)).pin_memory()
    pinX = torch.from_numpy(np.asfortranarray(P.X0)).pin_memory()
    outA = torch.empty((m0, m0), dtype=torch.complex128).pin_memory().t()
    outB = torch.empty((m0, m0), dtype=torch.complex128).pin_memory().t()
    h2d = pinA.numel() * 16 + (0 if pinB is None else pinB.numel() * 16) + pinX.numel() * 16
    d2h = 2 * m0 * m0 * 16

    def e2e_step():
        A.copy_(pinA, non_blocking=True)
        if pinB is not None:
            B.copy_(pinB, non_blocking=True)
        X.copy_(pinX, non_blocking=True)
        step()
        outA.copy_(Ah, non_blocking=True)
        outB.copy_(Bh, non_blocking=True)

    e2e_step()
    barrier()
    e0.record(stream)
    for _ in range(args.steps):
        e2e_step()
    e1.record(stream)
    barrier()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([e2e_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())

    # ---- full FEAST iterations (SURVEY §8(d) metric (1) "including the reduced eig"): projector,
    # node sum, orthonormalisation, reduced matrices, reduced eigenproblem (cuSOLVER), Ritz
    # vectors and residuals — feast_iterate through the public API, inputs resident.
    Xit = X.clone()
    f.iterate(A, B, Xit)
    barrier()
    n_it = max(1, min(3, args.steps))
    e0.record(f.stream)
    for _ in range(n_it):
        f.iterate(A, B, Xit)
    e1.record(f.stream)
    barrier()
    it_ms = e0.elapsed_time(e1) / n_it

    lu_solve, total = _flops(spec, n, m0, q)
    if rank == 0:
        proj_ms = sum(v["ms"] for k, v in prof.items()) / prof_steps  # kernel time per step
        line = {"metric": METRIC, "value": 1e3 / ms, "unit": "iter/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "complex128", "data": "synthetic",
                "config": {"workload": args.config, "n": n, "m0": m0, "q": q, "rule": "trapezoid(midpoint)",
                           "B": "I" if P.B is None else "I + 0.01 G_B/sqrt(n)", "mode": spec.mode,
                           "parallelism": f"nodes{world}", "nodes_per_rank": q // world,
                           "l2": "no flush: every step streams the q LU workspaces (>1 GB) through HBM, > 126 MB L2"},
                "lu_solve_tflops": lu_solve / (ms * 1e-3) / 1e12,
                "lu_solve_frac_peak": lu_solve / (ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS / world,
                "step_tflops": total / (ms * 1e-3) / 1e12,
                "clocks": clocks, "gpu_launches": gpu_launches,
                "e2e": {"value": 1e3 / e2e_ms, "unit": "iter/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
                "iteration_incl_reduced_eig": {"value": 1e3 / it_ms, "unit": "iter/s", "ms": it_ms,
                                               "what": "feast_iterate: projector + node sum + QR + reduced "
                                                       "matrices + reduced eig (cuSOLVER) + Ritz vectors/residuals"},
                "roofline": roofline}
        if world == 1 and not args.no_cpu_baseline:
            z, w, _, _ = f.nodes()
            line["cpu_baseline"] = cpu_baseline(args, P, np.array(z), np.array(w))
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
