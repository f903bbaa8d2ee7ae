#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_row_engines.py tests/test_gpu_block.py -q -m gpu -x > gpurun_out/pytest_rows5.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_rows5.log
rm -f gpurun_out/rs5.jsonl
for v in "policy - 72" "stream stg 72" "stream tma 100" "stream stg 100"; do set -- $v
E=$1; [ $E = policy ] && E=""; S=$2; [ $S = - ] && S=""
APL_ROW_ENGINE=$E APL_RS_STORE=$S APL_RS_BUDGET_KB=$3 timeout 300 python tools/block_ops_bench.py 2>&1 | grep "layernorm\|softmax" | sed "s/}$/, \"variant\": \"$1 $2 $3\"}/" >> gpurun_out/rs5.jsonl
done
echo ALLDONE
