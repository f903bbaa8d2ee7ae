"""Per-CTA phase timeline of one CTA-pair GEMM launch (apl_gemm_trace):
after warm-up, one traced launch of C[M,N] = A[M,K] B^T with a forced plan;
prints the median and max over CTAs of each phase's clock64 offset from the
CTA's entry (converted to us at the SM clock), and the spread of CTA start
times (%globaltimer).

    python tools/gemm_trace.py [--m 2048] [--n 1024] [--k 4096] [--bn 128]
"""
import argparse
import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2302_02599_b200 import _capi as A  # noqa: E402
from paper_2302_02599_b200.runtime import gemm  # noqa: E402

SLOTS = ["entry", "prologue_done", "pdl_wait_done", "producer_loop_entry", "issuer_loop_entry",
         "last_acc_committed", "last_acc_drained", "last_store_issued", "stores_done",
         "teardown", "exit"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=2048)
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--k", type=int, default=4096)
    ap.add_argument("--bn", type=int, default=128)
    args = ap.parse_args()
    lib = A.lib()
    a = torch.randn(args.m, args.k, device="cuda").bfloat16()
    bt = torch.randn(args.n, args.k, device="cuda").bfloat16()
    c = torch.empty(args.m, args.n, device="cuda", dtype=torch.bfloat16)
    assert lib.apl_gemm_force_plan(1, args.bn, 0) == 0
    for _ in range(5):
        gemm(a, bt, out=c)
    torch.cuda.synchronize()
    buf = torch.zeros(148 * 16, dtype=torch.int64, device="cuda")
    assert lib.apl_gemm_trace(buf.data_ptr(), buf.numel() * 8) == 0
    gemm(a, bt, out=c)
    torch.cuda.synchronize()
    lib.apl_gemm_trace(None, 0)
    lib.apl_gemm_force_plan(-1, -1, -1)
    t = buf.view(148, 16).cpu().tolist()
    ctas = [r for r in t if r[1] != 0]
    try:
        mhz = float(torch.cuda.clock_rate()) or 1965.0
    except Exception:
        mhz = 1965.0
    to_us = lambda cyc: cyc / mhz  # noqa: E731
    g0 = min(r[0] for r in ctas)
    out = {"shape": [args.m, args.n, args.k], "bn": args.bn, "ctas": len(ctas), "sm_mhz": mhz,
           "cta_start_spread_us": round((max(r[0] for r in ctas) - g0) / 1e3, 3), "phases": {}}
    for i, name in enumerate(SLOTS[1:], start=2):
        v = [to_us(r[i] - r[1]) for r in ctas if r[i] != 0]
        if v:
            out["phases"][name] = {"n": len(v), "median_us": round(statistics.median(v), 3),
                                   "max_us": round(max(v), 3)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
