#!/bin/bash
set -x
mkdir -p gpurun_out
APL_GEMM_PAIR=1 timeout 120 python -c "
import torch, sys
sys.path.insert(0, '.')
from paper_2302_02599_b200.runtime import gemm
for (m, n, k, lay) in [(256, 256, 64, 'nk'), (512, 512, 256, 'nk'), (1024, 768, 512, 'kn'), (300, 520, 200, 'nk')]:
    a = torch.randn(m, k, device='cuda').bfloat16(); bt = torch.randn(n, k, device='cuda').bfloat16()
    b = bt.t().contiguous() if lay == 'kn' else bt
    out = gemm(a, b, b_layout=lay); torch.cuda.synchronize()
    ref = a.double() @ bt.double().t()
    print(m, n, k, lay, ((out.double() - ref).abs().max() / ref.abs().max()).item(), flush=True)
" > gpurun_out/pair_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/pair_smoke.log
if grep -q "^300 520 200 nk" gpurun_out/pair_smoke.log; then
  APL_GEMM_PAIR=1 timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_executor.py -q -x > gpurun_out/pytest_pair.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_pair.log
  APL_GEMM_PAIR=1 timeout 600 python tools/gemm_bench.py > gpurun_out/gemm_bench_pair.json 2>&1
  APL_GEMM_PAIR=0 timeout 600 python tools/gemm_bench.py > gpurun_out/gemm_bench_single.json 2>&1
  timeout 600 python tools/mlp_bench.py > gpurun_out/mlp_bench.jsonl 2>&1
  APL_GEMM_PAIR=1 timeout 900 ncu --set full --clock-control none -k regex:gemm_bf16 -s 2 -c 1 -o gpurun_out/prof_gemm_pair python tools/gemm_bench.py --quick > gpurun_out/ncu_pair.log 2>&1
fi
echo ALLDONE
