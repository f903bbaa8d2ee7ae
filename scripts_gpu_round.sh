#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/gemm_bench.py > gpurun_out/gemm_bench.json 2>&1
timeout 600 python tools/mlp_bench.py > gpurun_out/mlp_bench.jsonl 2>&1
echo ALLDONE
