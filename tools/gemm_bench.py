"""Times the tcgen05 GEMM (libapl.so) on the config-5 shapes against
torch.matmul (cuBLAS) and the measured bf16 peak; prints one JSON object.

    python tools/gemm_bench.py [--quick]
    python tools/gemm_bench.py --sweep     # every launch plan per shape (JSON lines)
    python tools/gemm_bench.py --sweep --gelu --only "fc1"   # GELU epilogue, shape filter

--sweep forces each plan (apl_gemm_force_plan: 1-CTA / CTA-pair kernel,
N tile 128 / 256, whole tiles / stream-K) on every shape and prints one line
per (shape, plan) with its time, plus the automatic plan and cuBLAS.
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2302_02599_b200.runtime import gemm  # noqa: E402

# (name, M, N, K): GPT-2-medium MLP (x[16384,1024], W1[1024,4096], W2[4096,1024])
SHAPES = [
    ("fc1 full", 16384, 4096, 1024),
    ("fc2 full", 16384, 1024, 4096),
    ("fc1 split-m/8", 2048, 4096, 1024),
    ("fc2 split-m/8", 2048, 1024, 4096),
    ("fc1 split-n/8", 16384, 512, 1024),
    ("fc2 split-k/8", 16384, 1024, 512),
    ("square 8192", 8192, 8192, 8192),
]


def peak():
    p = ROOT / "MEASURED_PEAKS.json"
    return json.loads(p.read_text())["bf16_tflops"] if p.exists() else 1590.0


def time_fn(fn, iters):
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


def graph_time(fn, reps=20, repeats=5):
    """Best-of-`repeats` ms per call of `fn`, each repeat one CUDA-graph
    replay of `reps` back-to-back calls (no launch gaps, no Python)."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):  # the warm-up stream: its stream-K workspace exists
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(repeats):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / reps)
    return best


def sweep():
    import ctypes as C  # noqa: F401

    from paper_2302_02599_b200 import _capi as A

    lib = A.lib()
    pk = peak()
    plans = [("auto", -1, -1, -1)] + [
        (f"{'pair' if p else 'cta'}{bn}{'' if not sk else '-sk' if sk == 1 else f'-split{sk}'}",
         p, bn, sk)
        for p in (0, 1) for bn in (128, 256) for sk in (0, 1, 2, 4)]
    rounds = 3
    use_gelu = "--gelu" in sys.argv
    only = sys.argv[sys.argv.index("--only") + 1] if "--only" in sys.argv else ""
    for name, m, n, k in SHAPES:
        if only not in name:
            continue
        a = torch.randn(m, k, device="cuda").bfloat16()
        bt = torch.randn(n, k, device="cuda").bfloat16()
        c = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
        ref = a.float() @ bt.float().t()
        flops = 2.0 * m * n * k
        best = {}
        for _ in range(rounds):  # plans interleaved: clock drift hits every plan alike
            best["cublas"] = min(best.get("cublas", 1e30),
                                 graph_time(lambda: torch.matmul(a, bt.t(), out=c)))
            for pname, p, bn, sk in plans:
                assert lib.apl_gemm_force_plan(p, bn, sk) == 0
                best[pname] = min(best.get(pname, 1e30),
                                  graph_time(lambda: gemm(a, bt, out=c, gelu=use_gelu)))
        for pname, p, bn, sk in [("cublas", 0, 0, 0)] + plans:
            err = None
            if pname != "cublas":
                assert lib.apl_gemm_force_plan(p, bn, sk) == 0
                out = gemm(a, bt, out_dtype=torch.float32)
                err = ((out - ref).abs().max() / ref.abs().max()).item()
            ms = best[pname]
            print(json.dumps({"shape": name, "m": m, "n": n, "k": k, "plan": pname,
                              "epilogue": "gelu" if use_gelu and pname != "cublas" else "none",
                              "ms": round(ms, 4), "tflops": round(flops / ms / 1e9, 1),
                              "frac_of_peak": round(flops / ms / 1e9 / pk, 3),
                              "vs_cublas": round(best["cublas"] / ms, 3), "max_rel_err": err}),
                  flush=True)
        lib.apl_gemm_force_plan(-1, -1, -1)


def main():
    if "--sweep" in sys.argv:
        return sweep()
    quick = "--quick" in sys.argv
    shapes = SHAPES[:1] if quick else SHAPES
    out = {"peak_tflops": peak(), "rows": []}
    for name, m, n, k in shapes:
        a = torch.randn(m, k, device="cuda").bfloat16()
        bt = torch.randn(n, k, device="cuda").bfloat16()
        c = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
        flops = 2.0 * m * n * k
        iters = 3 if quick else 20
        # device time: CUDA-graph replays (best of 5), both sides alike -- the
        # per-call host cost (tensor-map encoding, ctypes; torch's dispatch)
        # is reported separately as the eager figures
        b_kn = bt.t().contiguous()
        fns = {"ours": lambda: gemm(a, bt, out=c),
               "gelu": lambda: gemm(a, bt, out=c, gelu=True),
               "kn": lambda: gemm(a, b_kn, out=c, b_layout="kn"),
               "cublas": lambda: torch.matmul(a, bt.t(), out=c)}
        dev = {k: min(graph_time(f) for _ in range(2)) for k, f in fns.items()}
        eager = {k: time_fn(fns[k], iters) for k in ("ours", "cublas")}
        ref = (a.float() @ bt.float().t())
        err = ((gemm(a, bt).float() - ref).abs().max() / ref.abs().max()).item()
        tf = lambda ms: round(flops / ms / 1e9, 1)  # noqa: E731
        out["rows"].append({
            "shape": name, "m": m, "n": n, "k": k,
            "ours_ms": round(dev["ours"], 4), "ours_tflops": tf(dev["ours"]),
            "ours_gelu_tflops": tf(dev["gelu"]), "ours_b_kn_tflops": tf(dev["kn"]),
            "cublas_ms": round(dev["cublas"], 4), "cublas_tflops": tf(dev["cublas"]),
            "ours_vs_cublas": round(dev["cublas"] / dev["ours"], 3),
            "ours_eager_tflops": tf(eager["ours"]), "cublas_eager_tflops": tf(eager["cublas"]),
            "frac_of_peak": round(flops / dev["ours"] / 1e9 / out["peak_tflops"], 3),
            "timing": "device: CUDA-graph replay of 20 back-to-back calls, best of 5 x 2; eager: "
                      "20 launches from Python",
            "max_rel_err": err})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
