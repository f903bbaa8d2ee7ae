#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -q -m gpu -x -k "convert or peer or capi" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
: > gpurun_out/runs.jsonl
for e in ldg bulk; do
  APL_COPY_ENGINE=$e timeout 300 python tools/run_probe.py 128 >> gpurun_out/runs.jsonl 2>&1
done
APL_SPLIT_RUN=100000000 PROBE_TAG=" splitall" timeout 300 python tools/run_probe.py 128 >> gpurun_out/runs.jsonl 2>&1
APL_SPLIT_RUN=100000000 PROBE_TAG=" splitall" timeout 300 python tools/run_probe.py 1024 >> gpurun_out/runs.jsonl 2>&1
timeout 600 python tools/size_probe.py > gpurun_out/probe_auto.jsonl 2> gpurun_out/probe_auto.err
APL_SPLIT_RUN=100000000 PROBE_TAG=" splitall" timeout 600 python tools/size_probe.py > gpurun_out/probe_split.jsonl 2> gpurun_out/probe_split.err
echo ALLDONE
