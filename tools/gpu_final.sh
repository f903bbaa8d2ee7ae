#!/bin/bash
# End-of-session evidence: smoke, bench (+ reference arm), launch list, ncu of
# the bench kernels and of the tile engine on the config-4 rank-3 conversion.
set -x
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-sweep > gpurun_out/bench_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:copy -s 6 -c 2 -o gpurun_out/ncu_bench_full python bench.py --steps 2 --warmup 3 --no-sweep > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:tile_copy -s 2 -c 1 -o gpurun_out/ncu_tile python tools/ncu_case.py 2,2,2 512,512,256 2 S0S1R RS1S0 > gpurun_out/ncu_tile.log 2>&1
echo ALLDONE
