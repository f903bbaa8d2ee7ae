# APL_SPLIT_RUN on the slow rank-3 classes with 128 B / 256 B runs
mkdir -p gpurun_out
out=gpurun_out/r3_split.jsonl; : > $out
for pr in "RS021R S01RS2" "RS12S0 S012RR" "RS1S02 S120RR" "RS012R S0RS21" "S2S10R RRS120" "RS0S2 RRS021"; do
  set -- $pr
  python tools/pair_probe.py 2,2,2 512,512,256 $1 $2 >> $out 2>&1
  for r in 128 256 512 1024; do APL_SPLIT_RUN=$r python tools/pair_probe.py 2,2,2 512,512,256 $1 $2 >> $out 2>&1; done
  APL_SPLIT_RUN=1024 APL_COPY_VARIANT=0 python tools/pair_probe.py 2,2,2 512,512,256 $1 $2 >> $out 2>&1
done
cat $out
