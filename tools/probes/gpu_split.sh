#!/bin/bash
# Split-descriptor check: GPU parity suite, then copy sweep with/without split rows.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
APL_SPLIT=1 timeout 600 python tools/copy_bench.py > gpurun_out/copy_split1.jsonl 2> gpurun_out/copy_split1.err
APL_SPLIT=0 timeout 600 python tools/copy_bench.py > gpurun_out/copy_split0.jsonl 2> gpurun_out/copy_split0.err
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo ALLDONE
