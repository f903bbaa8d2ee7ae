#!/bin/bash
# Block-op kernels: numerics, sanitizer, roofline with the prefetching row
# kernels on (default) and off (APL_ROW_PIPE=0).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_block.py tests/test_cpp_plan_executor.py -q -m gpu -x > gpurun_out/pytest_block.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_block.log
timeout 300 python tools/block_ops_bench.py > gpurun_out/block_ops_pipe.jsonl 2>&1
APL_ROW_PIPE=0 timeout 300 python tools/block_ops_bench.py > gpurun_out/block_ops_nopipe.jsonl 2>&1
timeout 1500 python -m pytest tests/test_gpu_sanitizer.py -q -m gpu > gpurun_out/pytest_sanitizer.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sanitizer.log
echo ALLDONE
