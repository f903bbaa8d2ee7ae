# Same-box A/B of two builds of libapl.so: ab/libapl_old.so and ab/libapl_new.so
# (built locally from the two source versions; ab/ is not tracked).
mkdir -p gpurun_out
for round in 1 2; do
  for v in old new; do
    cp ab/libapl_$v.so paper_2302_02599_b200/libapl.so
    python tools/gemm_bench.py > gpurun_out/ab_gemm_${v}_$round.json 2>&1
    python tools/mlp_bench.py > gpurun_out/ab_mlp_${v}_$round.jsonl 2>&1
    python -c "
import json
d=json.load(open('gpurun_out/ab_gemm_${v}_$round.json'))
print('$v', $round, [(r['shape'], r['ours_gelu_tflops']) for r in d['rows']])
m=[json.loads(l) for l in open('gpurun_out/ab_mlp_${v}_$round.jsonl')]
print('$v', $round, [(x['plan'], x['fuse'], x['graph_ms_per_train_step']) for x in m])
"
  done
done
