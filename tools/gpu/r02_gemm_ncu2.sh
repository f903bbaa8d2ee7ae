#!/bin/bash
mkdir -p gpurun_out
APL_GEMM_PAIR=1 APL_GEMM_BN=128 timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 3 -c 1 -o gpurun_out/ncu_pair128_fc2m python tools/gemm_case.py 2048 1024 4096 --iters 1 > gpurun_out/ncu_p1.log 2>&1
APL_GEMM_PAIR=1 APL_GEMM_BN=256 timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 3 -c 1 -o gpurun_out/ncu_pair256_sq python tools/gemm_case.py 8192 8192 8192 --iters 1 > gpurun_out/ncu_p2.log 2>&1
echo ALLDONE
