#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/split_probe.jsonl
for case in "2,2,2 512,512,256 S1S0R RRS120" "2,2,2 512,512,256 S10RR RRS210" "2,2,2 512,512,256 RS0S2 RRS021" "2,2,2 512,512,256 RRR RRS012" "2,2,2 512,512,256 RRR RS01S2" "2,2,2 512,512,256 S2RS1 S1S20R" "2,4 8192,8192 S01R RS01"; do
  for knob in "" "APL_SPLIT_RUN=128" "APL_SPLIT_RUN=256" "APL_SPLIT_RUN=1024" "APL_SPLIT_RUN=128 APL_COPY_VARIANT=0" "APL_SPLIT=0"; do
    env $knob timeout 120 python tools/pair_probe.py $case >> gpurun_out/split_probe.jsonl 2>> gpurun_out/split_probe.err
  done
done
echo ALLDONE
