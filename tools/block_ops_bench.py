"""HBM roofline of the block_ops.cu kernels at sizes well above L2 (inputs
>= 256 MiB, so every launch streams from HBM): achieved GB/s = algorithmic
bytes (each input read once + each output written once) / CUDA-event time,
against the measured copy peak in MEASURED_PEAKS.json.

    python tools/block_ops_bench.py
"""
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2302_02599_b200 import block_ops as B  # noqa: E402


def peak():
    try:
        m = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        for k in ("hbm_copy_gbs", "hbm_gbs", "copy_gbs"):
            if k in m:
                return float(m[k])
    except Exception:
        pass
    return 6542.4  # bench.py's measured copy peak (profiles/r01_bench.json)


def timed(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def main():
    pk = peak()
    rows, w = 131072, 1024  # 256 MiB of bf16
    x = torch.randn(rows, w, device="cuda").bfloat16()
    y = torch.empty_like(x)
    z = torch.randn(rows, w, device="cuda").bfloat16()
    g = torch.ones(w, device="cuda").bfloat16()
    m = (torch.rand(rows, w, device="cuda") < 0.5).to(torch.uint8)
    nb = x.numel() * 2
    cases = [
        ("layernorm", lambda: B.layernorm(x, g, g, y), 2 * nb),
        ("softmax", lambda: B.softmax(x, y), 2 * nb),
        ("masked_softmax (scale+u8 mask fused)", lambda: B.masked_softmax(x, y, 0.125, m, -1e4),
         2 * nb + m.numel()),
        ("add", lambda: B.add(x, z, y), 3 * nb),
        ("add u8 mask", lambda: B.add(x, m, y, -1e4), 2 * nb + m.numel()),
        ("scale", lambda: B.scale(x, y, 0.5), 2 * nb),
        ("transpose [128,1024,1024]", lambda: B.transpose_last2(x.view(128, 1024, 1024),
                                                                 y.view(128, 1024, 1024)), 2 * nb),
        ("layernorm backward (dx)", lambda: B.layernorm_backward(x, g, z, y), 3 * nb),
        ("softmax backward", lambda: B.softmax_backward(x, z, y), 3 * nb),
    ]
    table = torch.randn(50304, w, device="cuda").bfloat16()
    ids = torch.randint(0, 50304, (rows,), device="cuda", dtype=torch.int64)
    cases.append(("embedding lookup", lambda: B.embedding(ids, table, y), 2 * nb + ids.numel() * 8))
    blocks = [table[i * 6288:(i + 1) * 6288].contiguous() for i in range(8)]
    ptrs = [b.data_ptr() for b in blocks]
    cases.append(("embedding from 8 owner blocks", lambda: B.embedding_blocks(
        ids, ptrs, 8, 1, 50304, w, 0, y), 2 * nb + ids.numel() * 8))
    for name, fn, bytes_ in cases:
        ms = timed(fn)
        gbs = bytes_ / (ms * 1e-3) / 1e9
        print(json.dumps({"kernel": name, "engine": os.environ.get("APL_ROW_ENGINE", "stream"),
                          "ms": round(ms, 4), "algorithmic_bytes": bytes_,
                          "gbs": round(gbs, 1), "peak_gbs": pk, "frac": round(gbs / pk, 3)}),
              flush=True)


if __name__ == "__main__":
    main()
