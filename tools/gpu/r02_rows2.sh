#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_row_engines.py tests/test_gpu_block.py tests/test_plan_in_memory.py tests/test_gpu_backward.py tests/test_cpp_plan_executor.py -q -m gpu > gpurun_out/pytest_rows2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_rows2.log
timeout 300 python tools/block_ops_bench.py > gpurun_out/block_ops_policy.jsonl 2>&1
APL_ROW_ENGINE=stream timeout 300 python tools/block_ops_bench.py > gpurun_out/block_ops_stream2.jsonl 2>&1
APL_ROW_ENGINE=pipe timeout 300 python tools/block_ops_bench.py > gpurun_out/block_ops_pipe2.jsonl 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:row_stream -s 2 -c 1 -o gpurun_out/ncu_row_stream_ln python tools/block_ops_bench.py > gpurun_out/ncu_rows2.log 2>&1
echo ALLDONE
