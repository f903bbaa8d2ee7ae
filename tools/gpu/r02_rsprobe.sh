#!/bin/bash
mkdir -p gpurun_out
for b in 32 48 72 100 144 200; do
APL_ROW_ENGINE=stream APL_RS_BUDGET_KB=$b timeout 300 python tools/block_ops_bench.py 2>&1 | grep "layernorm\|softmax" | sed "s/}$/, \"budget_kb\": $b}/" >> gpurun_out/rs_budget.jsonl
done
echo ALLDONE
