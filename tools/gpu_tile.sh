#!/bin/bash
# Tile-engine check: parity with the engine forced, then run/size probes.
mkdir -p gpurun_out
APL_COPY_ENGINE=tile timeout 600 python -m pytest tests/test_gpu_convert.py tests/test_gpu_prepared.py -q -x > gpurun_out/pytest_tile.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tile.log
timeout 600 python -m pytest tests/test_gpu_convert.py tests/test_gpu_peer.py -q -x > gpurun_out/pytest_auto.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_auto.log
: > gpurun_out/tile_runs.jsonl
for e in tile ldg; do for mib in 128 1024; do
  APL_COPY_ENGINE=$e PROBE_TAG=" $e" timeout 300 python tools/run_probe.py $mib >> gpurun_out/tile_runs.jsonl 2>&1
done; done
timeout 300 python tools/size_probe.py > gpurun_out/probe_auto.jsonl 2>&1
echo ALLDONE
