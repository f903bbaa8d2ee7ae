#!/bin/bash
# Round-2 re-entry baseline: full GPU suite, smoke, bench (+ reference arm),
# GEMM shard-shape bench, block-op rooflines.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 python tools/gemm_bench.py > gpurun_out/gemm_bench.json 2> gpurun_out/gemm_bench.err
timeout 300 python tools/block_ops_bench.py > gpurun_out/block_ops_bench.jsonl 2>&1
echo ALLDONE
