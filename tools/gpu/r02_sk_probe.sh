#!/bin/bash
mkdir -p gpurun_out
for v in "0 128 0" "0 128 1" ; do set -- $v
APL_GEMM_PAIR=$1 APL_GEMM_BN=$2 APL_GEMM_STREAMK=$3 timeout 120 python tools/gemm_case.py 2048 1024 4096 --time --iters 50 2>&1 | head -1 | sed "s/}$/, \"plan\": \"$1-$2-$3\"}/" >> gpurun_out/sk_probe.jsonl
done
APL_SK_NOFIX=1 APL_GEMM_PAIR=0 APL_GEMM_BN=128 APL_GEMM_STREAMK=1 timeout 120 python tools/gemm_case.py 2048 1024 4096 --time --iters 50 2>&1 | head -1 | sed "s/}$/, \"plan\": \"sk-nofix\"}/" >> gpurun_out/sk_probe.jsonl
APL_GEMM_PAIR=0 APL_GEMM_BN=128 APL_GEMM_STREAMK=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_write.sum,dram__bytes_read.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_read.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active -k regex:gemm_bf16 -s 3 -c 1 python tools/gemm_case.py 2048 1024 4096 --iters 1 > gpurun_out/sk_ncu.txt 2>&1
APL_SK_NOFIX=1 APL_GEMM_PAIR=0 APL_GEMM_BN=128 APL_GEMM_STREAMK=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_write.sum,dram__bytes_read.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_read.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active -k regex:gemm_bf16 -s 3 -c 1 python tools/gemm_case.py 2048 1024 4096 --iters 1 >> gpurun_out/sk_ncu.txt 2>&1
echo ALLDONE
