#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/lock.jsonl
for ls in 0 1; do
  APL_COPY_LOCKSTEP=$ls PROBE_TAG=" lock=$ls" timeout 600 python tools/size_probe.py >> gpurun_out/lock.jsonl 2>> gpurun_out/lock.err
  APL_COPY_LOCKSTEP=$ls APL_COPY_ENGINE=ldg PROBE_TAG=" lock=$ls" timeout 600 python tools/run_probe.py 1024 >> gpurun_out/lock.jsonl 2>> gpurun_out/lock.err
done
echo ALLDONE
