#!/bin/bash
# bench.py at N>1 on a 1-GPU box: N processes share cuda:0 (functional check of the
# multi-rank peer path; the numbers share one GPU's HBM and are not NVLink numbers).
mkdir -p gpurun_out
for n in 2 4 8; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29600+n)) bench.py --gpus $n --steps 5 --warmup 3 > gpurun_out/bench_n$n.json 2> gpurun_out/bench_n$n.err
  echo "n=$n rc=$?"
done
echo ALLDONE
