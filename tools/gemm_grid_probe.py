"""Why the 256x256 pair tile is slow on small grids: time the forced pair256
plan on fc2 split-m/8 (2048x1024x4096: 32 clusters, one tile each), on two
such problems in one grouped launch (64 clusters), and on 4096x1024x4096
(64 clusters, one tile each), against cuBLAS; CUDA-graph device time."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))

import torch  # noqa: E402

from gemm_bench import graph_time  # noqa: E402
from paper_2302_02599_b200 import _capi as A  # noqa: E402
from paper_2302_02599_b200.runtime import gemm, gemm_grouped  # noqa: E402


def main():
    lib = A.lib()
    rows = []
    for plan in ((1, 256, 0), (0, 128, 0), (1, 128, 0)):
        lib.apl_gemm_force_plan(*plan)
        for m in (2048, 4096, 8192):
            a = torch.randn(m, 4096, device="cuda").bfloat16()
            bt = torch.randn(1024, 4096, device="cuda").bfloat16()
            c = torch.empty(m, 1024, device="cuda", dtype=torch.bfloat16)
            ms = min(graph_time(lambda: gemm(a, bt, out=c)) for _ in range(2))
            rows.append({"plan": plan, "shape": [m, 1024, 4096], "problems": 1,
                         "us": round(ms * 1e3, 2), "tflops": round(2 * m * 1024 * 4096 / ms / 1e9, 1)})
        a2 = [torch.randn(2048, 4096, device="cuda").bfloat16() for _ in range(2)]
        b2 = [torch.randn(4096, 1024, device="cuda").bfloat16() for _ in range(2)]
        c2 = [torch.empty(2048, 1024, device="cuda", dtype=torch.bfloat16) for _ in range(2)]
        fn = lambda: gemm_grouped([x.data_ptr() for x in a2], [x.data_ptr() for x in b2],  # noqa: E731
                                  [x.data_ptr() for x in c2], 1, 2048, 1024, 4096, 4096, 1024,
                                  1024, b_layout="kn")
        ms = min(graph_time(fn) for _ in range(2))
        rows.append({"plan": plan, "shape": [2048, 1024, 4096], "problems": 2,
                     "us": round(ms * 1e3, 2), "tflops": round(2 * 2 * 2048 * 1024 * 4096 / ms / 1e9, 1)})
    lib.apl_gemm_force_plan(-1, -1, -1)
    for m in (2048, 4096, 8192):
        a = torch.randn(m, 4096, device="cuda").bfloat16()
        bt = torch.randn(1024, 4096, device="cuda").bfloat16()
        c = torch.empty(m, 1024, device="cuda", dtype=torch.bfloat16)
        ms = min(graph_time(lambda: torch.matmul(a, bt.t(), out=c)) for _ in range(2))
        rows.append({"plan": "cublas", "shape": [m, 1024, 4096], "problems": 1,
                     "us": round(ms * 1e3, 2), "tflops": round(2 * m * 1024 * 4096 / ms / 1e9, 1)})
    for r in rows:
        print(json.dumps(r))


if __name__ == "__main__":
    main()
