"""Short-row all-to-all (S0R->RS0 on [8], runs of 64 B - 1 KiB) at 128 MiB -
1 GiB: TMA tensor tiles vs the LDG kernel's variants (env-forced per run),
CUDA-graph device time (profiles/r01_short_row_probe.jsonl).

    APL_COPY_ENGINE=tile|ldg [APL_COPY_VARIANT=1|3] python tools/short_row_probe.py
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
    tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("APL_COPY")) or "auto"
    for mib in (128, 512, 1024):
        for cols in (256, 512, 1024, 4096):
            rows = (mib << 20) // (2 * cols)
            r = conv_row([8], (rows, cols), 2, "S0R", "RS0", 6542.4)
            r["env"], r["mib"], r["run_bytes"] = tag, mib, cols * 2 // 8
            print(json.dumps(r), flush=True)
    r = conv_row([2, 2, 2], (512, 512, 256), 2, "S0S1R", "RS1S0", 6542.4)
    r["env"], r["mib"], r["run_bytes"] = tag, 128, 256
    print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
