#!/bin/bash
# Copy-engine change check: GPU parity suite + size probe (auto/ldg/bulk).
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/size_probe.py > gpurun_out/probe_auto.jsonl 2> gpurun_out/probe_auto.err
APL_COPY_ENGINE=ldg timeout 600 python tools/size_probe.py > gpurun_out/probe_ldg.jsonl 2> gpurun_out/probe_ldg.err
APL_COPY_ENGINE=bulk timeout 600 python tools/size_probe.py > gpurun_out/probe_bulk.jsonl 2> gpurun_out/probe_bulk.err
echo ALLDONE
