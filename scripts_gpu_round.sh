#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python tools/gemm_bench.py > gpurun_out/gemm_bench.json 2> gpurun_out/gemm_bench.err
timeout 600 python tools/mlp_bench.py > gpurun_out/mlp_bench.jsonl 2> gpurun_out/mlp_bench.err
timeout 600 python tools/copy_bench.py > gpurun_out/copy_auto.jsonl 2> gpurun_out/copy_auto.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 2 -c 2 -o gpurun_out/prof_gemm2 python tools/gemm_bench.py --quick > gpurun_out/ncu_gemm.log 2>&1
echo ALLDONE
