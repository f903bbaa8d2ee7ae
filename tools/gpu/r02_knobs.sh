#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/knobs.jsonl
for case in "2,4 8192,8192 S01R RS1" "2,4 8192,8192 RS10 S1R" "2,2,2 8192,8192 RS012 S01R" "2,4 8192,8192 RS0 RR" "2,2,2 8192,8192 S0S2 S21R" "2,2,2 512,512,256 S1S0R RRS120"; do
  for knob in "" "APL_COPY_VARIANT=0" "APL_COPY_VARIANT=1" "APL_COPY_VARIANT=2" "APL_COPY_VARIANT=3" "APL_COPY_LOCKSTEP=0" "APL_COPY_ENGINE=bulk" "APL_COPY_ENGINE=tile" "APL_COPY_CS=1" "APL_COPY_SPAN=1" "APL_COPY_VARIANT=1 APL_COPY_CTAS_PER_SM=8"; do
    env $knob timeout 120 python tools/pair_probe.py $case >> gpurun_out/knobs.jsonl 2>> gpurun_out/knobs.err
  done
done
echo ALLDONE
