#!/bin/bash
# Round-2 evidence: full GPU suite, smoke, bench (+ reference arm), GEMM
# bench, block ops, MLP / block timings, launch list, stamped ncu traffic.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_gpu_final.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_final.log
timeout 600 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_final.json 2> gpurun_out/bench_ref_final.err
timeout 600 python tools/gemm_bench.py > gpurun_out/gemm_bench_final.json 2> gpurun_out/gemm_bench_final.err
timeout 300 python tools/block_ops_bench.py > gpurun_out/block_ops_final.jsonl 2>&1
timeout 600 python tools/mlp_bench.py > gpurun_out/mlp_bench_final.jsonl 2>&1
timeout 600 python tools/block_bench.py > gpurun_out/block_bench_final.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu > gpurun_out/bench_ncu_final.log 2>&1
timeout 900 python tools/ncu_traffic.py > gpurun_out/ncu_traffic_final.log 2>&1

timeout 900 ncu --set full --clock-control none -k regex:"box_copy|bulk_copy" -s 6 -c 2 --csv --page details python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu > gpurun_out/ncu_bench_details.csv 2> gpurun_out/ncu_bench_details.err
echo ALLDONE2
