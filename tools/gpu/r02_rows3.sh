#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_row_engines.py tests/test_gpu_block.py -q -m gpu -x > gpurun_out/pytest_rows3.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_rows3.log
rm -f gpurun_out/rs3.jsonl
for v in "stream tma 72" "stream tma 100" "stream stg 72" "pipe tma 72"; do set -- $v
APL_ROW_ENGINE=$1 APL_RS_STORE=$2 APL_RS_BUDGET_KB=$3 timeout 300 python tools/block_ops_bench.py 2>&1 | grep "layernorm\|softmax" | sed "s/}$/, \"store\": \"$2\", \"budget_kb\": $3}/" >> gpurun_out/rs3.jsonl
done
timeout 300 python tools/block_ops_bench.py > gpurun_out/block_ops_policy3.jsonl 2>&1
echo ALLDONE
