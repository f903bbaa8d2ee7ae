#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -q -m gpu -x -k "convert or peer or capi" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
: > gpurun_out/runs.jsonl
for e in ldg bulk; do
  APL_COPY_ENGINE=$e timeout 300 python tools/run_probe.py 128 >> gpurun_out/runs.jsonl 2>&1
  APL_COPY_ENGINE=$e timeout 300 python tools/run_probe.py 1024 >> gpurun_out/runs.jsonl 2>&1
  for sl in 4 16; do APL_SLABS=$sl APL_COPY_ENGINE=$e timeout 300 python -c "
import sys,json; sys.path.insert(0,'tools'); sys.path.insert(0,'.')
from size_probe import conv_row
pk=json.load(open('MEASURED_PEAKS.json'))['hbm_gbs']
for m,sh in (([2],(8192,8192)),([8],(8192,8192))):
    print(json.dumps(conv_row(m,sh,2,'S0R','RS0',pk,tag=' slabs=$sl')),flush=True)
" >> gpurun_out/runs.jsonl 2>&1; done
done
timeout 600 python tools/size_probe.py > gpurun_out/probe_auto.jsonl 2> gpurun_out/probe_auto.err
echo ALLDONE
