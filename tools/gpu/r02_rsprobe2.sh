#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/rs_policy.jsonl
for pol in 0 1 2 3; do for b in 72 100; do
APL_ROW_ENGINE=stream APL_RS_POLICY=$pol APL_RS_BUDGET_KB=$b timeout 300 python tools/block_ops_bench.py 2>&1 | grep "layernorm\|softmax" | sed "s/}$/, \"budget_kb\": $b, \"policy\": $pol}/" >> gpurun_out/rs_policy.jsonl
done; done
echo ALLDONE
