set -x
timeout 300 python tools/peer_loopback.py --ranks 8 > gpurun_out/r02_peer_loopback_8.jsonl 2> gpurun_out/r02_peer_loopback_8.err; echo rc=$?
cat gpurun_out/r02_peer_loopback_8.jsonl; tail -5 gpurun_out/r02_peer_loopback_8.err
timeout 300 python tools/peer_loopback.py --ranks 4 > gpurun_out/r02_peer_loopback_4.jsonl 2> gpurun_out/r02_peer_loopback_4.err; echo rc=$?
cat gpurun_out/r02_peer_loopback_4.jsonl; tail -5 gpurun_out/r02_peer_loopback_4.err
