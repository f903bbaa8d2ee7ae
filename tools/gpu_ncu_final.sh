#!/bin/bash
# ncu evidence for the current kernels: bench launch list, full captures of the
# bench's two conversion kernels, the backward (MN-major A) GEMM, write/read probes.
mkdir -p gpurun_out
timeout 300 python tools/write_probe.py > gpurun_out/write_probe.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-sweep > gpurun_out/bench_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:copy -s 6 -c 2 -o gpurun_out/ncu_bench_full python bench.py --steps 2 --warmup 3 --no-sweep > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:gemm -s 2 -c 3 -o gpurun_out/ncu_gemm_bwd python -m pytest tests/test_gpu_backward.py -q -k "single_device and 1024" > gpurun_out/ncu_gemm_bwd.log 2>&1
echo ALLDONE
