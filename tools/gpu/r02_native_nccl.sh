#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_cpp_plan_executor.py -q -m gpu -k "distributed or general" > gpurun_out/pytest_native_nccl.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_native_nccl.log
echo ALLDONE
