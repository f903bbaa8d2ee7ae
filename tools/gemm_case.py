"""One GEMM shape, launched a few times (for ncu captures and A/B timing of
the GEMM knobs).

    python tools/gemm_case.py M N K [--iters 5] [--gelu] [--time]

--time prints {"shape", "ms", "tflops"} from CUDA events over --iters
back-to-back launches (after 3 warm-up launches), like tools/gemm_bench.py.
"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2302_02599_b200.runtime import gemm  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("m", type=int)
    ap.add_argument("n", type=int)
    ap.add_argument("k", type=int)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--gelu", action="store_true")
    ap.add_argument("--time", action="store_true")
    ap.add_argument("--cublas", action="store_true")
    a = ap.parse_args()
    torch.manual_seed(0)
    x = torch.randn(a.m, a.k, device="cuda").bfloat16()
    bt = torch.randn(a.n, a.k, device="cuda").bfloat16()
    c = torch.empty(a.m, a.n, device="cuda", dtype=torch.bfloat16)
    fn = (lambda: torch.matmul(x, bt.t(), out=c)) if a.cublas else \
        (lambda: gemm(x, bt, out=c, gelu=a.gelu))
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(a.iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / a.iters
    if a.time:
        print(json.dumps({"shape": [a.m, a.n, a.k], "cublas": a.cublas, "gelu": a.gelu,
                          "ms": round(ms, 4),
                          "tflops": round(2.0 * a.m * a.n * a.k / ms / 1e9, 1)}))
    ref = x.float() @ bt.float().t()
    out = gemm(x, bt, out_dtype=torch.float32)
    err = ((out - ref).abs().max() / ref.abs().max()).item()
    assert err < 1e-2, err


if __name__ == "__main__":
    main()
