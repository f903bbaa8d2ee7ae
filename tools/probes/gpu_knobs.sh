#!/bin/bash
# Copy-engine knob sweep at 128 MiB / 1 GiB (A2A, config 3/4 cases).
mkdir -p gpurun_out
out=gpurun_out/knobs.jsonl; : > $out
for eng in ldg bulk; do for spread in 0 1; do
  APL_COPY_ENGINE=$eng APL_COPY_SPREAD=$spread PROBE_TAG=" spread=$spread" timeout 300 python tools/size_probe.py --quick >> $out 2>>gpurun_out/knobs.err
done; done
for v in 0 1 2; do for spread in 0 1; do
  APL_COPY_ENGINE=ldg APL_COPY_VARIANT=$v APL_COPY_SPREAD=$spread PROBE_TAG=" v=$v spread=$spread" timeout 300 python tools/size_probe.py --quick >> $out 2>>gpurun_out/knobs.err
done; done
for c in 2 4 6 8; do
  APL_COPY_ENGINE=ldg APL_COPY_CTAS_PER_SM=$c PROBE_TAG=" v=3 ctas=$c" timeout 300 python tools/size_probe.py --quick >> $out 2>>gpurun_out/knobs.err
done
echo ALLDONE
