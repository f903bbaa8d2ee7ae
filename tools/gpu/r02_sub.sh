#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_backward.py -q -m gpu -x > gpurun_out/pytest_sub.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sub.log
timeout 600 python tools/gemm_grid_probe.py > gpurun_out/grid_probe_sub.jsonl 2> gpurun_out/grid_probe_sub.err
echo ALLDONE
