set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_nccl.py -x -q -p no:cacheprovider > gpurun_out/r02_nccl.log 2>&1; echo nccl_rc=$?
tail -30 gpurun_out/r02_nccl.log
timeout 600 python bench.py --gpus 1 --steps 10 --warmup 3 > gpurun_out/r02_b1.json 2> gpurun_out/r02_b1.err; echo b1_rc=$?
timeout 600 python bench.py --gpus 4 --steps 5 --warmup 3 --no-sweep > gpurun_out/r02_b4.json 2> gpurun_out/r02_b4.err; echo b4_rc=$?
timeout 600 python bench.py --gpus 2 --transport nccl --steps 3 --warmup 3 --no-sweep > gpurun_out/r02_b2nccl.json 2> gpurun_out/r02_b2nccl.err; echo b2n_rc=$?
tail -c 1500 gpurun_out/r02_b4.err; tail -c 1500 gpurun_out/r02_b2nccl.err
