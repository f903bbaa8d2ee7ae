"""`apl_convert` is the reference CLI's `plan convert` (proj/tools/
plan_main.cpp:98-109 options, 179-202 output) on the drop-in layout API:
the printed steps must be the reference's golden paths, errors must map to
the CLI's exit codes (plan_main.cpp:256-265), and --execute (GPU) must
round-trip bit-exactly."""
import gzip
import json
import random
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
CLI = ROOT / "paper_2302_02599_b200" / "apl_convert"
KIND = {0: "all-gather", 1: "all-reduce", 2: "reduce-scatter", 3: "all-to-all", 4: "shard-slice"}

pytestmark = pytest.mark.skipif(not CLI.exists(), reason="apl_convert not built")


def run(*args, timeout=120):
    return subprocess.run([str(CLI), *args], capture_output=True, text=True, timeout=timeout)


def test_cli_paths_equal_reference_golden_paths():
    with gzip.open(ROOT / "tests" / "golden" / "paths.json.gz", "rt") as f:
        cases = json.load(f)["cases"]
    rng = random.Random(7)
    checked = 0
    for case in cases:
        mesh = "x".join(map(str, case["mesh"]))
        shape = "x".join(map(str, case["shape"]))
        for src, tgt, steps, _cost, _n in rng.sample(case["pairs"], min(12, len(case["pairs"]))):
            r = run("--from", src, "--to", tgt, "--mesh", mesh, "--shape", shape,
                    "--dtype-bytes", str(case["dtype_bytes"]))
            assert r.returncode == 0, r.stderr
            lines = r.stdout.splitlines()
            assert lines[0].startswith(f"{src} -> {tgt}: {len(steps)} step(s), ")
            cur = src
            for line, (kind, dim, tdim, axis, result) in zip(lines[1:], steps):
                want = f"  {KIND[kind]} dim {dim}" + (f" -> dim {tdim}" if tdim >= 0 else "") + \
                    f" axis {axis}: {cur} -> {result}"
                assert line == want
                cur = result
            checked += 1
    assert checked > 100


def test_cli_error_exit_codes():
    assert run("--from", "S9R", "--to", "RR", "--mesh", "2x2", "--shape", "8x8").returncode == 3
    assert run("--from", "S0R", "--to", "RR", "--mesh", "2x2", "--shape", "7x8").returncode == 3


@pytest.mark.gpu
@pytest.mark.parametrize("args", [
    ["--from", "S0R", "--to", "RS0", "--mesh", "2x2", "--shape", "1024x1024"],
    ["--from", "S01R", "--to", "S1S0", "--mesh", "2x4", "--shape", "8192x8192", "--dtype-bytes", "2"],
    ["--from", "S012R", "--to", "RS012", "--mesh", "2x2x2", "--shape", "8192x8192",
     "--dtype-bytes", "2", "--stepwise"],
])
def test_cli_execute_round_trip(cuda, args):
    r = run(*args, "--execute", "--iters", "3")
    assert r.returncode == 0, r.stdout + r.stderr
    assert re.search(r"round trip bit-exact", r.stdout), r.stdout
