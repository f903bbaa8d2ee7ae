#!/bin/bash
mkdir -p gpurun_out
APL_DEBUG=1 APL_GEMM_PAIR=1 APL_GEMM_BN=256 timeout 120 python tools/gemm_case.py 8192 8192 8192 --time --iters 10 > gpurun_out/mc2_quick.log 2>&1
APL_DEBUG=1 APL_GEMM_MC=0 APL_GEMM_PAIR=1 APL_GEMM_BN=256 timeout 120 python tools/gemm_case.py 8192 8192 8192 --time --iters 10 >> gpurun_out/mc2_quick.log 2>&1
timeout 900 python tools/gemm_bench.py --sweep > gpurun_out/gemm_sweep_mc2.jsonl 2> gpurun_out/gemm_sweep_mc2.err
APL_GEMM_MC=0 timeout 900 python tools/gemm_bench.py --sweep > gpurun_out/gemm_sweep_nomc2.jsonl 2> gpurun_out/gemm_sweep_nomc2.err
echo ALLDONE
