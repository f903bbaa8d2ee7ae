set -x
timeout 1500 python -m pytest tests/test_gpu_peer.py tests/test_gpu_peer_executor.py tests/test_gpu_peer_block.py -q -p no:cacheprovider --durations=10 > gpurun_out/r02_peer_tests.log 2>&1; echo rc=$?
tail -25 gpurun_out/r02_peer_tests.log
for n in 2 4 8; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29611 tools/peer_latency.py > gpurun_out/r02_peer_latency_n$n.jsonl 2> gpurun_out/r02_peer_latency_n$n.err; echo lat_rc=$?
cat gpurun_out/r02_peer_latency_n$n.jsonl; tail -5 gpurun_out/r02_peer_latency_n$n.err
done
