#!/bin/bash
mkdir -p gpurun_out
S="2048 1024 4096"
APL_GEMM_PAIR=1 APL_GEMM_BN=256 APL_GEMM_STREAMK=1 timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 3 -c 1 -o gpurun_out/ncu_sk_pair256 python tools/gemm_case.py $S --iters 1 > gpurun_out/ncu_sk1.log 2>&1
APL_GEMM_PAIR=1 APL_GEMM_BN=256 APL_GEMM_STREAMK=0 timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 3 -c 1 -o gpurun_out/ncu_pair256 python tools/gemm_case.py $S --iters 1 > gpurun_out/ncu_sk2.log 2>&1
timeout 300 ncu --set full --clock-control none -s 3 -c 1 -o gpurun_out/ncu_cublas_fc2m python tools/gemm_case.py $S --iters 1 --cublas > gpurun_out/ncu_sk3.log 2>&1
APL_GEMM_PAIR=0 APL_GEMM_BN=128 APL_GEMM_STREAMK=0 timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 3 -c 1 -o gpurun_out/ncu_cta128 python tools/gemm_case.py $S --iters 1 > gpurun_out/ncu_sk4.log 2>&1
echo ALLDONE
