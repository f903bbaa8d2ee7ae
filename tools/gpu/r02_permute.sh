#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_permute.py tests/test_cpp_plan_executor.py tests/test_gpu_block.py tests/test_plan_in_memory.py -q -m gpu > gpurun_out/pytest_permute.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_permute.log
echo ALLDONE
