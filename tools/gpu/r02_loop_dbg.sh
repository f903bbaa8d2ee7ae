#!/bin/bash
mkdir -p gpurun_out
timeout 120 python tools/peer_loopback.py --ranks 2 --iters 20 --debug > gpurun_out/loop_dbg.jsonl 2> gpurun_out/loop_dbg.err
APL_PULL_GRID_CAP=8 timeout 120 python tools/peer_loopback.py --ranks 2 --iters 20 --debug > gpurun_out/loop_dbg2.jsonl 2> gpurun_out/loop_dbg2.err
echo ALLDONE
