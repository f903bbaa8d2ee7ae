# Knob sweep on the slowest rank-3 2x2x2 classes with 256 B / 128 B runs
# (profiles/r02_pairs_222_r3_all.jsonl): engine, LDG variant, CTAs per SM.
mkdir -p gpurun_out
out=gpurun_out/r3_knobs.jsonl; : > $out
for pr in "RS021R S01RS2" "RS12S0 S012RR" "RS1S02 S120RR" "RS012R S0RS21" "S0S1R RS1S0" "RRR RRS01"; do
  set -- $pr
  python tools/pair_probe.py 2,2,2 512,512,256 $1 $2 >> $out 2>&1
  for e in ldg bulk tile; do APL_COPY_ENGINE=$e python tools/pair_probe.py 2,2,2 512,512,256 $1 $2 >> $out 2>&1; done
  for v in 0 1 2 3; do APL_COPY_ENGINE=ldg APL_COPY_VARIANT=$v python tools/pair_probe.py 2,2,2 512,512,256 $1 $2 >> $out 2>&1; done
  for c in 2 4 8; do APL_COPY_ENGINE=ldg APL_COPY_CTAS_PER_SM=$c python tools/pair_probe.py 2,2,2 512,512,256 $1 $2 >> $out 2>&1; done
done
cat $out
