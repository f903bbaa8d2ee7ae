set -x
timeout 1500 python -m pytest tests/test_gpu_exhaustive.py tests/test_gpu_peer.py -q -p no:cacheprovider --durations=20 > gpurun_out/r02_parity.log 2>&1; echo rc=$?
tail -40 gpurun_out/r02_parity.log
