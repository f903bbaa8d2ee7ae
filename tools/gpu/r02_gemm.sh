#!/bin/bash
# GEMM plans: correctness of every plan, the plan sweep, block ops with the
# occupancy-sized pipe grids, sanitizer, batched-strategy backward, subset
# peer all-reduce.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py -q -m gpu -x > gpurun_out/pytest_gemm.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gemm.log
timeout 600 python tools/gemm_bench.py --sweep > gpurun_out/gemm_sweep.jsonl 2> gpurun_out/gemm_sweep.err
timeout 300 python tools/block_ops_bench.py > gpurun_out/block_ops_pipe3.jsonl 2>&1
APL_ROW_PIPE=0 timeout 300 python tools/block_ops_bench.py > gpurun_out/block_ops_nopipe3.jsonl 2>&1
timeout 1500 python -m pytest tests/test_gpu_block.py tests/test_gpu_sanitizer.py tests/test_gpu_backward.py -q -m gpu > gpurun_out/pytest_block3.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_block3.log
timeout 900 python -m pytest tests/test_gpu_peer.py -q -m gpu -k "subset or fused_gemm" > gpurun_out/pytest_peer.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_peer.log
echo ALLDONE
