"""DRAM traffic of the dominant kernel (zgemm_dmma_kernel) per launch vs its algorithmic bytes.

Two passes over the SAME bench step (project (+ left) + reduce of --config=Ck, serialised profile
mode, the launch sequence bench.py's roofline pass times):

    python tools/zgemm_traffic.py alg  gpurun_out/zg_alg.json     # algorithmic bytes / flops
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        -k regex:zgemm_dmma --profile-from-start off --csv --log-file gpurun_out/zg_ncu.csv \
        python tools/zgemm_traffic.py ncu
    python tools/zgemm_traffic.py merge gpurun_out/zg_alg.json gpurun_out/zg_ncu.csv profiles/zgemm_traffic.json

ncu flushes L2 before every replayed launch (--cache-control all), so the DRAM bytes are the
cold-cache figure: every operand tile the kernel touches comes from HBM once if the tiling
re-reads nothing."""
import csv
import json
import sys

sys.path.insert(0, ".")


def run_step(mode, config, batch=0):
    import numpy as np
    import torch
    import synth
    from paper_1404_2891_b200 import Feast, empty_colmajor, feast as fb
    spec = synth.CONFIGS[config]
    bi = spec.mode == "bi"
    if spec.n >= 4096:
        P = synth.make_pencil_torch(config)
        A, B, X = P.A, P.B, P.X0
        P.V = P.lam = None
    else:
        P = synth.make_pencil(config)
        d = lambda a: None if a is None else torch.from_numpy(np.asfortranarray(a)).to("cuda")
        A, B, X = d(P.A), d(P.B), d(P.X0)
    n, m0, s = P.n, P.m0, spec
    V = fb.colmajor(torch.linalg.solve(X.conj().T @ X, X.conj().T).conj().T) if bi else None
    del P
    torch.cuda.empty_cache()
    f = Feast(n, m0, s.c, s.r, s.aspect, s.n_e, s.rule, fb.BI if bi else fb.RIGHT, B is None, max_batch=batch)
    Q = empty_colmajor(n, m0)
    QL = empty_colmajor(n, m0) if bi else None
    Ah = empty_colmajor(m0, m0)
    Bh = empty_colmajor(m0, m0)

    def step():
        if bi:
            f.project_bi(A, B, X, V, Q, QL)
        else:
            f.project(A, B, X, Q)
        f.reduce(A, B, Q, QL, Ah, Bh)

    f.profile(True, serial=True)
    step()                      # warm-up: lazy init, workspace, kernel attributes
    torch.cuda.synchronize()
    f.profile(True, serial=True)
    if mode == "ncu":
        torch.cuda.profiler.start()
    step()
    torch.cuda.synchronize()
    if mode == "ncu":
        torch.cuda.profiler.stop()
    zg = f.profile_summary()["zgemm"]
    f.profile(False)
    return zg


def merge(alg_path, ncu_path, out_path, config):
    alg = json.load(open(alg_path))
    rows = []
    with open(ncu_path) as fh:
        lines = [l for l in fh if l.startswith('"')]
    for r in csv.DictReader(lines):
        if "zgemm_dmma" not in r["Kernel Name"]:
            continue
        rows.append(r)
    per = {}
    for r in rows:
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
                 "msecond": 1e6}.get(unit, 1)
        per.setdefault(r["ID"], {})[r["Metric Name"]] = v * scale
    n = len(per)
    dram = sum(m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0) for m in per.values())
    rd = sum(m.get("dram__bytes_read.sum", 0) for m in per.values())
    ns = sum(m.get("gpu__time_duration.sum", 0) for m in per.values())
    out = {
        "config": config,
        "kernel": "zgemm_dmma_kernel",
        "launches": n,
        "launches_alg": alg["launches"],
        "dram_bytes_per_launch": dram / n,
        "dram_read_bytes_per_launch": rd / n,
        "algorithmic_bytes_per_launch": alg["bytes"] / alg["launches"],
        "traffic_over_algorithmic": dram / alg["bytes"] if alg["bytes"] else None,
        "ncu_cold_cache_ms_per_step": ns * 1e-6,
        "ncu_tflops_cold_serialised": alg["flops"] / (ns * 1e-9) / 1e12 if ns else None,
        "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                  f"--clock-control none -k regex:zgemm_dmma over one serialised {config} bench step "
                  "(tools/zgemm_traffic.py)",
    }
    json.dump(out, open(out_path, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    mode = sys.argv[1]
    cfg = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--config=")), "C2")
    batch = int(next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--batch=")), "0"))
    args = [a for a in sys.argv[2:] if not a.startswith("--")]
    if mode == "alg":
        zg = run_step("alg", cfg)
        json.dump(zg, open(args[0], "w"), indent=1)
        print(zg)
    elif mode == "ncu":
        run_step("ncu", cfg, batch)
    elif mode == "merge":
        merge(args[0], args[1], args[2], cfg)
