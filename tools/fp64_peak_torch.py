"""cuBLAS FP64 yardsticks (DGEMM, ZGEMM) burst and sustained, timed with CUDA events.
Complements tools/fp64_peak.cu (DMMA/DFMA microbenchmark). Writes JSON lines to stdout."""
import json, time, torch

def bench(dtype, n, secs=None, reps=10):
    a = torch.randn(n, n, dtype=dtype, device="cuda"); b = torch.randn(n, n, dtype=dtype, device="cuda")
    c = a @ b; torch.cuda.synchronize()
    fl = (8 if dtype.is_complex else 2) * n ** 3
    best = 0.0
    if secs is None:
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); torch.matmul(a, b, out=c); e1.record(); e1.synchronize()
            best = max(best, fl / (e0.elapsed_time(e1) * 1e-3) / 1e12)
        return best
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k = 0; t0 = time.time(); e0.record()
    while time.time() - t0 < secs:
        torch.matmul(a, b, out=c); k += 1
        if k % 4 == 0: torch.cuda.synchronize()
    e1.record(); e1.synchronize()
    return fl * k / (e0.elapsed_time(e1) * 1e-3) / 1e12

for dt, n in [(torch.float64, 8192), (torch.complex128, 4096), (torch.complex128, 8192)]:
    print(json.dumps({"kind": f"cublas_{dt}", "n": n, "burst_tflops": round(bench(dt, n), 3),
                      "sustained_tflops": round(bench(dt, n, secs=4.0), 3)}), flush=True)
