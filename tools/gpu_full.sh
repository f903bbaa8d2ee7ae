#!/bin/bash
# Full GPU check: parity suite, smoke, headline bench (+ reference arm), config-2 sweep,
# size probe, ncu launch list and a full capture of the bench's dominant kernel.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 python tools/copy_bench.py --sweep > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err
timeout 600 python tools/size_probe.py > gpurun_out/probe_auto.jsonl 2> gpurun_out/probe_auto.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/bench_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:copy -s 6 -c 2 -o gpurun_out/ncu_bench_full python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_full.log 2>&1
echo ALLDONE
