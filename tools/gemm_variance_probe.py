"""fc1 split-m/8 (2048x4096x1024) run-to-run check: one process, every plan
and cuBLAS timed three times (CUDA-graph replays, tools/gemm_bench.graph_time),
buffer addresses printed. Run it in several fresh processes.

    for i in 1 2 3 4 5 6; do python tools/gemm_variance_probe.py; done
"""
import sys, json
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / 'tools'))
import torch
from gemm_bench import graph_time
from paper_2302_02599_b200 import _capi as A
from paper_2302_02599_b200.runtime import gemm
lib = A.lib()
m, n, k = 2048, 4096, 1024
a = torch.randn(m, k, device="cuda").bfloat16(); bt = torch.randn(n, k, device="cuda").bfloat16()
c = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
res = {"ptrs": [hex(a.data_ptr()), hex(bt.data_ptr()), hex(c.data_ptr())]}
for name, plan in (("auto", (-1, -1, -1)), ("pair256", (1, 256, 0)), ("cta256", (0, 256, 0)), ("pair128", (1, 128, 0))):
    lib.apl_gemm_force_plan(*plan)
    res[name] = [round(2.0*m*n*k/graph_time(lambda: gemm(a, bt, out=c))/1e9, 1) for _ in range(3)]
lib.apl_gemm_force_plan(-1, -1, -1)
res["cublas"] = [round(2.0*m*n*k/graph_time(lambda: torch.matmul(a, bt.t(), out=c))/1e9, 1) for _ in range(3)]
print(json.dumps(res))
