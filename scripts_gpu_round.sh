#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python tools/copy_bench.py --sweep > gpurun_out/copy_sweep.jsonl 2> gpurun_out/copy_sweep.err
timeout 600 python tools/copy_bench.py > gpurun_out/copy_auto.jsonl 2> gpurun_out/copy_auto.err
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python tools/mlp_bench.py > gpurun_out/mlp_bench.jsonl 2> gpurun_out/mlp_bench.err
echo ALLDONE
