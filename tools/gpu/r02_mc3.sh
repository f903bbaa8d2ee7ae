#!/bin/bash
mkdir -p gpurun_out
APL_GEMM_MC=1 timeout 1500 python tools/gemm_bench.py --sweep > gpurun_out/gemm_sweep_mc3.jsonl 2> gpurun_out/gemm_sweep_mc3.err
echo ALLDONE
