#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_peer.py -q -m gpu -k "push or epochs" > gpurun_out/pytest_push.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_push.log
timeout 1200 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_backward.py tests/test_gpu_convert.py -q -m gpu -x > gpurun_out/pytest_gemm_copy.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gemm_copy.log
timeout 600 python tools/gemm_bench.py > gpurun_out/gemm_bench_graph.json 2> gpurun_out/gemm_bench_graph.err
timeout 900 python tools/pair_sweep.py --mesh 2,4 --shape 8192,8192 > gpurun_out/pairs_2x4_v3.jsonl 2> gpurun_out/pairs_2x4_v3.err
timeout 900 python tools/pair_sweep.py --mesh 2,2,2 --shape 8192,8192 > gpurun_out/pairs_222_r2_v3.jsonl 2> gpurun_out/pairs_222_r2_v3.err
timeout 600 python bench.py --steps 30 --no-cpu > gpurun_out/bench_v3.json 2> gpurun_out/bench_v3.err
echo ALLDONE
