#!/bin/bash
# Quick check: GEMM + convert GPU tests, headline bench, config-2 sweep.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/ -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python tools/copy_bench.py --sweep > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err
timeout 600 python tools/gemm_bench.py > gpurun_out/gemm_bench.json 2> gpurun_out/gemm_bench.err
echo ALLDONE
