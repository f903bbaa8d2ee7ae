#!/bin/bash
# One GPU session: parity tests, smoke, bench (copy variants A/B), launch list, ncu captures.
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/ -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
for v in 0 1; do APL_COPY_VARIANT=$v timeout 600 python bench.py > gpurun_out/bench_v$v.json 2> gpurun_out/bench_v$v.err; done
timeout 600 python tools/gemm_bench.py > gpurun_out/gemm_bench.json 2> gpurun_out/gemm_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:box_copy -s 6 -c 2 -o gpurun_out/prof_box_copy python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 2 -c 2 -o gpurun_out/prof_gemm python tools/gemm_bench.py --quick > gpurun_out/ncu_gemm.log 2>&1
echo ALLDONE
