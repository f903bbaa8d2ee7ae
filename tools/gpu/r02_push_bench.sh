#!/bin/bash
mkdir -p gpurun_out
timeout 300 python bench.py --gpus 4 --steps 5 --warmup 3 --no-sweep --transport push > gpurun_out/bench_n4_push.json 2> gpurun_out/bench_n4_push.err
timeout 300 python bench.py --gpus 4 --steps 5 --warmup 3 --no-sweep > gpurun_out/bench_n4_pull.json 2> gpurun_out/bench_n4_pull.err
timeout 900 python tools/pair_sweep.py --mesh 2,2,2 --shape 8192,8192 > gpurun_out/pairs_222_r2_v4.jsonl 2> gpurun_out/pairs_222_r2_v4.err
timeout 1200 python tools/pair_sweep.py --mesh 2,2,2 --shape 512,512,256 --sample 600 > gpurun_out/pairs_222_r3_v4.jsonl 2> gpurun_out/pairs_222_r3_v4.err
timeout 900 python tools/pair_sweep.py --mesh 2,4 --shape 8192,8192 > gpurun_out/pairs_2x4_v4.jsonl 2> gpurun_out/pairs_2x4_v4.err
echo ALLDONE
