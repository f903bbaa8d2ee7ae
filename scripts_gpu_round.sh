#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
APL_GEMM_PAIR=0 timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x > gpurun_out/pytest_single.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_single.log
timeout 600 python tools/gemm_bench.py > gpurun_out/gemm_bench.json 2>&1
timeout 600 python tools/mlp_bench.py > gpurun_out/mlp_bench.jsonl 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --set full --clock-control none -k regex:gemm_bf16 -s 2 -c 1 -o gpurun_out/prof_gemm_pair python tools/gemm_bench.py --quick > gpurun_out/ncu_pair.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"box_copy|bulk_copy" -s 6 -c 2 -o gpurun_out/prof_bench python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_bench.log 2>&1
echo ALLDONE
