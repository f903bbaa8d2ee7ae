#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_gemm.py -q -m gpu -x > gpurun_out/pytest_splitk.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_splitk.log
timeout 1500 python tools/gemm_bench.py --sweep > gpurun_out/gemm_sweep_split.jsonl 2> gpurun_out/gemm_sweep_split.err
timeout 600 python tools/gemm_bench.py > gpurun_out/gemm_bench_split.json 2> gpurun_out/gemm_bench_split.err
echo ALLDONE
