"""C++ callers of the reference layout API build against include/ + libapl.so
unchanged (tests/cpp/drop_in_test.cpp)."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def test_cpp_drop_in_compiles_links_and_runs(tmp_path):
    exe = tmp_path / "drop_in"
    lib = ROOT / "paper_2302_02599_b200"
    cmd = ["g++", "-std=c++20", "-O1", f"-I{ROOT / 'include'}", str(ROOT / "tests/cpp/drop_in_test.cpp"),
           f"-L{lib}", "-lapl", f"-Wl,-rpath,{lib}", "-o", str(exe)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    try:
        import torch

        gpu = torch.cuda.is_available()
    except Exception:
        gpu = False
    r = subprocess.run([str(exe)] + (["--gpu"] if gpu else []), capture_output=True, text=True,
                       timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "drop-in ok" in r.stdout
