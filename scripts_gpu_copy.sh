#!/bin/bash
mkdir -p gpurun_out
for v in 0 1 2 3; do APL_COPY_VARIANT=$v timeout 600 python tools/copy_bench.py > gpurun_out/copy_v$v.jsonl 2> gpurun_out/copy_v$v.err; done
APL_COPY_VARIANT=0 APL_COPY_CTAS_PER_SM=4 timeout 600 python tools/copy_bench.py > gpurun_out/copy_v0_g4.jsonl 2>&1
timeout 600 ncu --set full --clock-control none -k regex:box_copy -s 9 -c 3 -o gpurun_out/prof_copy_sweep python tools/copy_bench.py --quick > gpurun_out/ncu_copy.log 2>&1
