"""Write-only and read-only HBM bandwidth on one B200 (the AG fan-out is
8 bytes written per byte read, so its roofline is closer to the write-only
rate than to the copy rate). Graph-timed fill_ / sum over 1 GiB."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))

import torch  # noqa: E402

from size_probe import graph_ms  # noqa: E402


def main():
    n = 1 << 29  # bf16 elements = 1 GiB
    x = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    y = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    ms_w = graph_ms(lambda st: x.fill_(1.0))
    ms_c = graph_ms(lambda st: y.copy_(x))
    ms_r = graph_ms(lambda st: x.sum(dtype=torch.float32))
    gb = 2 * n
    print(json.dumps({"write_only_gbs": round(gb / ms_w / 1e6, 1),
                      "copy_gbs": round(2 * gb / ms_c / 1e6, 1),
                      "read_only_gbs": round(gb / ms_r / 1e6, 1)}))


if __name__ == "__main__":
    main()
