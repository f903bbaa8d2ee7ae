#!/bin/bash
# Size dependence of the copy engines + ncu captures of the config-3/4 kernels.
set -x
mkdir -p gpurun_out
timeout 600 python tools/size_probe.py > gpurun_out/probe_auto.jsonl 2> gpurun_out/probe_auto.err
APL_COPY_ENGINE=ldg timeout 600 python tools/size_probe.py > gpurun_out/probe_ldg.jsonl 2> gpurun_out/probe_ldg.err
APL_COPY_ENGINE=bulk timeout 600 python tools/size_probe.py > gpurun_out/probe_bulk.jsonl 2> gpurun_out/probe_bulk.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:copy -s 2 -c 1 -o gpurun_out/ncu_s012r python tools/ncu_case.py 2,2,2 8192,8192 2 S012R RS012 > gpurun_out/ncu_s012r.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:copy -s 2 -c 1 -o gpurun_out/ncu_s01r_s1s0 python tools/ncu_case.py 2,4 8192,8192 2 S01R S1S0 > gpurun_out/ncu_s01r.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:copy -s 2 -c 1 -o gpurun_out/ncu_a2a128 python tools/ncu_case.py 8 8192,8192 2 S0R RS0 > gpurun_out/ncu_a2a128.log 2>&1
echo ALLDONE
