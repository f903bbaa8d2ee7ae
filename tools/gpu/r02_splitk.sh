#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_gemm.py -q -m gpu -x > gpurun_out/pytest_splitk2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_splitk2.log
timeout 1500 python tools/gemm_bench.py --sweep > gpurun_out/gemm_sweep_split2.jsonl 2> gpurun_out/gemm_sweep_split2.err
timeout 600 python tools/gemm_bench.py > gpurun_out/gemm_bench_split2.json 2> gpurun_out/gemm_bench_split2.err
echo ALLDONE
