"""bench.py keeps the driver's contract at N = 1 and N > 1 (ranks spawned by
bench.py itself, sharing the GPU here) for every transport, and the
reference arm prints its line: one JSON line each, the keys the driver
reads, sane values. Short runs; the numbers are not checked, the shape is."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
pytestmark = pytest.mark.gpu

KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
        "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "roofline",
        "gpu_launches", "clocks", "e2e"}


def _line(args, timeout=900):
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_n1(cuda):
    d = _line(["--steps", "3", "--warmup", "3", "--no-sweep", "--no-cpu"])
    assert KEYS <= set(d) and d["n_gpus"] == 1 and d["value"] > 0
    assert d["roofline"]["bound"] == "hbm" and 0 < d["roofline"]["frac"] <= 1.2
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0


@pytest.mark.parametrize("transport", ["peer", "push", "nccl"])
def test_bench_n2_every_transport(cuda, transport):
    d = _line(["--gpus", "2", "--steps", "2", "--warmup", "3", "--no-sweep", "--no-cpu",
               "--transport", transport])
    assert KEYS <= set(d) and d["n_gpus"] == 2 and d["value"] > 0
    assert d["unit"] == "GB/s per GPU"


def test_bench_reference_arm(cuda):
    d = _line(["--impl", "reference", "--steps", "1", "--warmup", "3"])
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["cores"] >= 1 and d["e2e"]["h2d_bytes_per_step"] == 0
