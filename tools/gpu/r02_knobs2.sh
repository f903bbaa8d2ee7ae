#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/knobs2.jsonl
for case in "8 65536,8192 S0R RR" "8 65536,8192 S0R RS0" "2,4 8192,8192 S01R RR" "2,4 8192,8192 S01R RS0" "2,4 8192,8192 S1R RR" "2,2,2 8192,8192 S012R RS012" "2,2,2 512,512,256 S0S1R RS1S0" "2,2,2 8192,8192 S0R RR"; do
  for knob in "" "APL_COPY_VARIANT=0" "APL_COPY_VARIANT=1" "APL_COPY_VARIANT=2" "APL_COPY_VARIANT=3"; do
    env $knob timeout 120 python tools/pair_probe.py $case >> gpurun_out/knobs2.jsonl 2>> gpurun_out/knobs2.err
  done
done
echo ALLDONE
