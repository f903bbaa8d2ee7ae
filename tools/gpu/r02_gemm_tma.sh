#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_backward.py tests/test_gpu_executor.py tests/test_gpu_block.py tests/test_gpu_sanitizer.py tests/test_gpu_prepared.py -q -m gpu -x > gpurun_out/pytest_gemm_tma.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gemm_tma.log
timeout 900 python tools/gemm_bench.py --sweep > gpurun_out/gemm_sweep_tma.jsonl 2> gpurun_out/gemm_sweep_tma.err
APL_GEMM_TMA_OUT=0 timeout 600 python tools/gemm_bench.py > gpurun_out/gemm_bench_stg.json 2> gpurun_out/gemm_bench_stg.err
echo ALLDONE
