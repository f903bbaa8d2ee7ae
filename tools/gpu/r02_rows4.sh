#!/bin/bash
mkdir -p gpurun_out
APL_ROW_ENGINE=stream timeout 600 ncu --set full --clock-control none --import-source on -k regex:row_stream -s 2 -c 1 -o gpurun_out/ncu_rs_ln_tma python tools/block_ops_bench.py > gpurun_out/ncu_a.log 2>&1
APL_ROW_ENGINE=stream timeout 600 ncu --set full --clock-control none --import-source on -k regex:row_stream -s 25 -c 1 -o gpurun_out/ncu_rs_sm_tma python tools/block_ops_bench.py > gpurun_out/ncu_b.log 2>&1
echo ALLDONE
