#!/bin/bash
mkdir -p gpurun_out
for n in 2 4 8; do
timeout 200 python tools/peer_loopback.py --ranks $n --modes fused > gpurun_out/loop_fused_$n.jsonl 2> gpurun_out/loop_fused_$n.err
timeout 200 python tools/peer_loopback.py --ranks $n --modes unfused > gpurun_out/loop_unfused_$n.jsonl 2> gpurun_out/loop_unfused_$n.err
done
echo ALLDONE
