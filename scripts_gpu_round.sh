#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
APL_COPY_ENGINE=ldg timeout 900 python -m pytest tests/test_gpu_convert.py -q -x > gpurun_out/pytest_gpu_ldg.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_ldg.log
APL_COPY_ENGINE=bulk timeout 900 python -m pytest tests/test_gpu_convert.py -q -x > gpurun_out/pytest_gpu_bulk.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_bulk.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
for e in ldg bulk; do APL_COPY_ENGINE=$e timeout 600 python tools/copy_bench.py > gpurun_out/copy_$e.jsonl 2> gpurun_out/copy_$e.err; done
timeout 900 python tools/copy_bench.py --sweep > gpurun_out/copy_sweep.jsonl 2> gpurun_out/copy_sweep.err
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python tools/mlp_bench.py > gpurun_out/mlp_bench.jsonl 2> gpurun_out/mlp_bench.err
timeout 900 ncu --set full --clock-control none -k regex:bulk_copy -s 6 -c 2 -o gpurun_out/prof_bulk python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_bulk.log 2>&1
echo ALLDONE
