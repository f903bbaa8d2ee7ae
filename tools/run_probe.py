"""A2A S0R->RS0 at a fixed global size with varying run lengths and mesh
sizes (simulated on one B200): does the contiguous run length or the piece
count set the achieved HBM fraction?

    python tools/run_probe.py [MiB]
"""
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))

from size_probe import conv_row  # noqa: E402


def main():
    import json as _j
    peak = _j.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
    mib = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    if "--skew" in sys.argv:
        rows = (mib << 20) // (2 * 8192)
        for skew in (None, 0, 2048, 6144, 8192, 65536 + 2048, 1 << 20, (1 << 20) + 6144):
            r = conv_row([8], (rows, 8192), 2, "S0R", "RS0", peak, tag=f" skew={skew}", skew=skew)
            print(json.dumps(r), flush=True)
        return
    for p in (2, 4, 8):
        for run in (512, 1024, 2048, 4096, 8192, 16384):
            cols = run * p // 2
            rows = (mib << 20) // (2 * cols)
            if rows % p or rows < p:
                continue
            r = conv_row([p], (rows, cols), 2, "S0R", "RS0", peak, tag=f" run={run}" + os.environ.get("PROBE_TAG", ""))
            print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
