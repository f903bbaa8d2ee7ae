#!/bin/bash
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/clocks_sweep.csv &
SMI=$!
timeout 900 python tools/gemm_bench.py --sweep > gpurun_out/gemm_sweep2.jsonl 2> gpurun_out/gemm_sweep2.err
kill $SMI
timeout 900 python -m pytest tests/test_gpu_block.py tests/test_gpu_sanitizer.py tests/test_plan_in_memory.py -q -m gpu -k "batched_matmul_strategy or sanitizer or memcheck or racecheck or in_memory" > gpurun_out/pytest_fix.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fix.log
timeout 900 python -m pytest tests/test_gpu_peer.py -q -m gpu -k "subset" > gpurun_out/pytest_peer2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_peer2.log
echo ALLDONE
