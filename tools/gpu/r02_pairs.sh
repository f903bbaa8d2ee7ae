#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_permute.py -q -m gpu -k plans > gpurun_out/pytest_permute2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_permute2.log
timeout 900 python tools/pair_sweep.py --mesh 2,4 --shape 8192,8192 > gpurun_out/pairs_2x4.jsonl 2> gpurun_out/pairs_2x4.err
timeout 900 python tools/pair_sweep.py --mesh 2,2,2 --shape 8192,8192 > gpurun_out/pairs_222_r2.jsonl 2> gpurun_out/pairs_222_r2.err
timeout 1200 python tools/pair_sweep.py --mesh 2,2,2 --shape 512,512,256 --sample 600 > gpurun_out/pairs_222_r3.jsonl 2> gpurun_out/pairs_222_r3.err
echo ALLDONE
