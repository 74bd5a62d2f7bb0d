"""bench.py's launcher contract on CPU (no GPU, no hot path: --dry-run): `--gpus N` without an
outer torchrun spawns N ranks itself (torch.distributed.run, gloo here), the max-over-ranks
reduction runs, and rank 0 prints n_gpus = N; a WORLD_SIZE that disagrees with --gpus fails."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          env=e, timeout=300, cwd=ROOT)


@pytest.mark.parametrize("n", [1, 2])
def test_bench_spawns_its_own_ranks(n):
    r = _run(["--gpus", str(n), "--dry-run"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1                      # rank 0 alone prints
    assert lines[0]["n_gpus"] == n and lines[0]["max_rank_time"] == float(n)


def test_bench_rejects_world_mismatch():
    r = _run(["--gpus", "2", "--dry-run"], env={"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode == 2 and "WORLD_SIZE=1 != --gpus 2" in r.stderr


def test_bench_default_config_is_c4():
    import bench
    import synth
    assert bench.DEFAULT_CONFIG == "C4" and synth.CONFIGS["C4"].mode == "bi"
    lu, total = bench._flops(synth.CONFIGS["C4"], 16384, 512, 32)
    # C4 4.47e14 flop per iteration (incl. left solves)
    assert abs(total - 4.47e14) / 4.47e14 < 0.01
