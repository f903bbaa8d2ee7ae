#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_executor.py -q -x > gpurun_out/pytest_gemm.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gemm.log
APL_GEMM_PAIR=0 timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_executor.py -q -x > gpurun_out/pytest_gemm_single.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gemm_single.log
timeout 600 python tools/mlp_bench.py > gpurun_out/mlp_bench.jsonl 2>&1
APL_FUSED_AR=0 timeout 600 python tools/mlp_bench.py --quick > gpurun_out/mlp_bench_nofuse.jsonl 2>&1
echo ALLDONE
