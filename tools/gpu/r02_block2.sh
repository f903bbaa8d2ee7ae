#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_block.py tests/test_gpu_sanitizer.py tests/test_cpp_plan_executor.py -q -m gpu > gpurun_out/pytest_block2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_block2.log
timeout 300 python tools/block_ops_bench.py > gpurun_out/block_ops_pipe2.jsonl 2>&1
# GEMM: timing per shape and knob, then ncu of the split shapes
for s in "2048 4096 1024" "2048 1024 4096" "16384 512 1024" "16384 1024 512"; do
  python tools/gemm_case.py $s --time --iters 50 >> gpurun_out/gemm_knobs.jsonl 2>&1
  python tools/gemm_case.py $s --time --iters 50 --cublas >> gpurun_out/gemm_knobs.jsonl 2>&1
  APL_GEMM_PAIR=1 python tools/gemm_case.py $s --time --iters 50 | sed 's/}$/, "knob": "pair=1"}/' >> gpurun_out/gemm_knobs.jsonl 2>&1
  APL_GEMM_PAIR=0 python tools/gemm_case.py $s --time --iters 50 | sed 's/}$/, "knob": "pair=0"}/' >> gpurun_out/gemm_knobs.jsonl 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 3 -c 1 -o gpurun_out/ncu_gemm_fc1_splitm python tools/gemm_case.py 2048 4096 1024 --iters 1 > gpurun_out/ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 3 -c 1 -o gpurun_out/ncu_gemm_fc2_splitm python tools/gemm_case.py 2048 1024 4096 --iters 1 > gpurun_out/ncu2.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:nvjet\|gemm\|Kernel -s 3 -c 1 -o gpurun_out/ncu_cublas_fc2_splitm python tools/gemm_case.py 2048 1024 4096 --iters 1 --cublas > gpurun_out/ncu3.log 2>&1
echo ALLDONE
