#!/bin/bash
mkdir -p gpurun_out
for f in "1 128" "1 256"; do set -- $f
APL_GEMM_PAIR=$1 APL_GEMM_BN=$2 APL_GEMM_STREAMK=0 timeout 120 python tools/gemm_case.py 2048 1024 4096 --time --iters 20 >> gpurun_out/mc_quick.log 2>&1; echo "rc=$? pair=$1 bn=$2" >> gpurun_out/mc_quick.log
APL_GEMM_MC=0 APL_GEMM_PAIR=$1 APL_GEMM_BN=$2 APL_GEMM_STREAMK=0 timeout 120 python tools/gemm_case.py 2048 1024 4096 --time --iters 20 >> gpurun_out/mc_quick.log 2>&1; echo "rc=$? nomc pair=$1 bn=$2" >> gpurun_out/mc_quick.log
done
grep -q "rc=0 pair=1 bn=128" gpurun_out/mc_quick.log || { echo ABORT; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_backward.py tests/test_gpu_executor.py tests/test_gpu_block.py tests/test_gpu_sanitizer.py tests/test_gpu_prepared.py -q -m gpu -x > gpurun_out/pytest_gemm_mc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gemm_mc.log
timeout 900 python tools/gemm_bench.py --sweep > gpurun_out/gemm_sweep_mc.jsonl 2> gpurun_out/gemm_sweep_mc.err
echo ALLDONE
