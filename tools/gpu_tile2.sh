#!/bin/bash
mkdir -p gpurun_out
APL_COPY_ENGINE=tile timeout 600 python -m pytest tests/test_gpu_convert.py tests/test_gpu_prepared.py -q > gpurun_out/pytest_tile.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tile.log
timeout 900 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
echo ALLDONE
