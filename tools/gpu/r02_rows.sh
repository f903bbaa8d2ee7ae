#!/bin/bash
# TMA-streamed row engine: parity (both engines byte-identical), block tests,
# the three re-entry failures, HBM rooflines of both engines, GEMM plans.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_row_engines.py tests/test_gpu_block.py tests/test_plan_in_memory.py tests/test_gpu_sanitizer.py -q -m gpu -x > gpurun_out/pytest_rows.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_rows.log
timeout 600 python -m pytest tests/test_gpu_peer.py -q -m gpu -k "subsets" > gpurun_out/pytest_subsets.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_subsets.log
timeout 300 python tools/block_ops_bench.py > gpurun_out/block_ops_stream.jsonl 2>&1
APL_ROW_ENGINE=pipe timeout 300 python tools/block_ops_bench.py > gpurun_out/block_ops_pipe.jsonl 2>&1
timeout 600 python tools/gemm_bench.py > gpurun_out/gemm_bench2.json 2> gpurun_out/gemm_bench2.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:row_stream -s 2 -c 2 -o gpurun_out/ncu_row_stream python tools/block_ops_bench.py > gpurun_out/ncu_rows.log 2>&1
echo ALLDONE
