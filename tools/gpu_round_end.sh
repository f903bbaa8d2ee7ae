#!/bin/bash
# Round-end evidence in one call: full GPU suite, smoke, bench + reference arm,
# config-2 sweep, MLP bench, transformer-block bench / gradient check / kernel
# rooflines, launch list, ncu of the bench kernels.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 python tools/copy_bench.py --sweep > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err
timeout 600 python tools/mlp_bench.py > gpurun_out/mlp_bench.jsonl 2>&1
timeout 600 python tools/block_bench.py > gpurun_out/block_bench.jsonl 2>&1
timeout 600 python tools/block_grad_check.py 2>/dev/null | grep '^{' > gpurun_out/block_grads.jsonl
timeout 300 python tools/block_ops_bench.py > gpurun_out/block_ops_bench.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-sweep > gpurun_out/bench_ncu.log 2>&1
echo ALLDONE
