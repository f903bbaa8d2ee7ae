#!/bin/bash
# Mid-round evidence after the row-engine and GEMM changes.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_gpu_mid.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_mid.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_mid.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_mid.log
timeout 600 python bench.py > gpurun_out/bench_mid.json 2> gpurun_out/bench_mid.err
timeout 600 python tools/gemm_bench.py > gpurun_out/gemm_bench_mid.json 2> gpurun_out/gemm_bench_mid.err
timeout 300 python tools/block_ops_bench.py > gpurun_out/block_ops_mid.jsonl 2>&1
timeout 600 python tools/mlp_bench.py > gpurun_out/mlp_bench_mid.jsonl 2>&1
timeout 600 python tools/block_bench.py > gpurun_out/block_bench_mid.jsonl 2>&1
for n in 2 4 8; do timeout 300 python tools/peer_loopback.py --ranks $n > gpurun_out/peer_loopback_$n.jsonl 2> gpurun_out/peer_loopback_$n.err; done
echo ALLDONE
