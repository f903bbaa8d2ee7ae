#!/bin/bash
mkdir -p gpurun_out
timeout 120 python tools/gemm_case.py 2048 1024 4096 --time --iters 20 > gpurun_out/prod_quick.log 2>&1 || { echo ABORT; cat gpurun_out/elect_quick.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_backward.py tests/test_gpu_executor.py tests/test_gpu_block.py tests/test_gpu_sanitizer.py tests/test_gpu_prepared.py -q -m gpu -x > gpurun_out/pytest_gemm_prod.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gemm_elect.log
timeout 900 python tools/gemm_bench.py --sweep > gpurun_out/gemm_sweep_prod.jsonl 2> gpurun_out/gemm_sweep_prod.err
echo ALLDONE
