"""Engine / variant crossover at small and mid sizes (launch-bound regime):
for each case and global size, the device time of every copy engine / LDG
variant forced by env (run once per setting, see gpu script), CUDA-graph
timed like size_probe.py.

    APL_COPY_ENGINE=... APL_COPY_VARIANT=... python tools/crossover_probe.py
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
    peak = 6542.4
    tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("APL_COPY"))
    for mib in (1, 4, 16, 32, 64, 128, 256):
        for cols, a, b in ((1024, "S0R", "RR"), (1024, "S0R", "RS0"), (8192, "S0R", "RS0")):
            rows = (mib << 20) // (2 * cols)
            r = conv_row([8], (rows, cols), 2, a, b, peak)
            r["env"] = tag or "auto"
            r["mib"] = mib
            print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
