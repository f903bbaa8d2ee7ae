"""Where a one-tile-per-CTA GEMM spends its time: device time (CUDA-graph
replays, tools/gemm_bench.graph_time) of C[M,N] = A[M,K] B^T for a sweep of
K at fixed M, N, for forced launch plans and cuBLAS, with a least-squares
line time = overhead + K/64 * per_kblock. The slope is the mainloop rate (ns
per 64-deep K block per tile); the intercept is the fixed cost (launch,
prologue, pipeline fill, epilogue).

    python tools/gemm_k_slope.py [--m 2048] [--n 1024] [--ks 512,1024,2048,4096,8192]
"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))

import torch  # noqa: E402

from gemm_bench import graph_time  # noqa: E402
from paper_2302_02599_b200 import _capi as A  # noqa: E402
from paper_2302_02599_b200.runtime import gemm  # noqa: E402

PLANS = {"cta128": (0, 128, 0), "pair128": (1, 128, 0), "auto": (-1, -1, -1)}


def fit(xs, ys):
    n = len(xs)
    mx, my = sum(xs) / n, sum(ys) / n
    sxx = sum((x - mx) ** 2 for x in xs)
    slope = sum((x - mx) * (y - my) for x, y in zip(xs, ys)) / sxx
    return my - slope * mx, slope


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=2048)
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--ks", default="512,1024,2048,4096,8192")
    args = ap.parse_args()
    ks = [int(k) for k in args.ks.split(",")]
    lib = A.lib()
    times = {p: [] for p in list(PLANS) + ["cublas"]}
    for k in ks:
        a = torch.randn(args.m, k, device="cuda").bfloat16()
        bt = torch.randn(args.n, k, device="cuda").bfloat16()
        c = torch.empty(args.m, args.n, device="cuda", dtype=torch.bfloat16)
        best = {}
        for _ in range(3):  # interleaved rounds, best of each
            best["cublas"] = min(best.get("cublas", 1e30),
                                 graph_time(lambda: torch.matmul(a, bt.t(), out=c)))
            for p, (pair, bn, sk) in PLANS.items():
                assert lib.apl_gemm_force_plan(pair, bn, sk) == 0
                best[p] = min(best.get(p, 1e30), graph_time(lambda: gemm(a, bt, out=c)))
        lib.apl_gemm_force_plan(-1, -1, -1)
        for p, ms in best.items():
            times[p].append(ms * 1e3)
            print(json.dumps({"m": args.m, "n": args.n, "k": k, "plan": p, "us": round(ms * 1e3, 3),
                              "tflops": round(2.0 * args.m * args.n * k / ms / 1e9, 1)}),
                  flush=True)
    xs = [k / 64 for k in ks]
    for p, ys in times.items():
        b0, b1 = fit(xs, ys)
        print(json.dumps({"plan": p, "fit": "us = overhead + kblocks * per_kblock",
                          "overhead_us": round(b0, 3), "per_kblock_ns": round(1e3 * b1, 2)}),
              flush=True)


if __name__ == "__main__":
    main()
