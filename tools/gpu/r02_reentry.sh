#!/bin/bash
# Round-2 re-entry: full GPU suite, smoke, bench (+ reference arm), GEMM
# shard shapes (auto plan + every forced plan), block-op rooflines, launch list,
# peer latency on 2/4/8 ranks sharing the GPU.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 1500 python -m pytest tests/ -q -m gpu --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 python tools/gemm_bench.py > gpurun_out/gemm_bench.json 2> gpurun_out/gemm_bench.err
timeout 900 python tools/gemm_bench.py --sweep > gpurun_out/gemm_sweep.jsonl 2> gpurun_out/gemm_sweep.err
timeout 300 python tools/block_ops_bench.py > gpurun_out/block_ops_bench.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-sweep > gpurun_out/bench_ncu.log 2>&1
for n in 2 4 8; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29611 tools/peer_latency.py > gpurun_out/peer_latency_n$n.jsonl 2> gpurun_out/peer_latency_n$n.err
done
timeout 300 python bench.py --gpus 4 --steps 5 --warmup 3 --no-sweep > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err
echo ALLDONE
