#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/gemm_grid_probe.py > gpurun_out/grid_probe_krot.jsonl 2> gpurun_out/grid_probe_krot.err
APL_GEMM_KROT=0 timeout 600 python tools/gemm_grid_probe.py > gpurun_out/grid_probe_nokrot.jsonl 2> gpurun_out/grid_probe_nokrot.err
echo ALLDONE
