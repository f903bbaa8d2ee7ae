"""compute-sanitizer over every kernel family (memory/race
checking). tools/sanitize_case.py runs small, self-checking invocations of
the copy engines, the tcgen05 GEMMs, the block ops and the fused peer
exchange; each runs in a subprocess under memcheck (and racecheck for the
shared-memory-staged kernels) and must report zero errors."""
import os
import shutil
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


def _run(tool, case, env_extra=None, timeout=900):
    env = dict(os.environ)
    env["APL_DEBUG"] = "1"  # a failing launch says which step failed
    env.update(env_extra or {})
    cmd = [SAN, "--tool", tool, "--error-exitcode", "9", "--print-limit", "20",
           sys.executable, str(ROOT / "tools" / "sanitize_case.py"), case]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
    out = p.stdout + p.stderr
    assert p.returncode == 0, out[-4000:]
    assert f"sanitize case {case}: ok" in out, out[-4000:]
    clean = ("RACECHECK SUMMARY: 0 hazards displayed (0 errors, 0 warnings)" if tool == "racecheck"
             else "ERROR SUMMARY: 0 errors")
    assert clean in out, out[-4000:]
    return out


@pytest.mark.parametrize("engine", ["ldg", "bulk", "tile"])
def test_memcheck_copy_engines(cuda, engine):
    _run("memcheck", "copies", {"APL_COPY_ENGINE": engine})


def test_memcheck_gemm(cuda):
    _run("memcheck", "gemm")


@pytest.mark.parametrize("engine", ["policy", "stream", "pipe"])
def test_memcheck_block_ops(cuda, engine):
    """every row op on each row engine (stream: TMA slabs, TMA-store
    write-back for the softmaxes)"""
    _run("memcheck", "block", {} if engine == "policy" else {"APL_ROW_ENGINE": engine})


def test_memcheck_peer_exchange(cuda):
    _run("memcheck", "peer", {"CUDA_DEVICE_MAX_CONNECTIONS": "32"})


@pytest.mark.parametrize("case,env", [("block", {}), ("block", {"APL_ROW_ENGINE": "stream"}),
                                      ("copies", {"APL_COPY_ENGINE": "bulk"})])
def test_racecheck_shared_memory(cuda, case, env):
    _run("racecheck", case, env)
