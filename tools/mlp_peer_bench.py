"""BASELINE config 5 on N GPUs over peer memory (one process per GPU):
the GPT-2-medium MLP with the pinned Megatron selection -- fc1 split-n:0
(local tcgen05 GEMM + GELU on each rank's W1 column block), fc2 split-k:0
(GEMM + all-reduce fused over peer memory: the epilogue scatters fp32 row
blocks to their owners, owners reduce and store into every rank). Prints one
JSON line (rank 0): ms per forward (max over ranks) and TFLOP/s of the whole
job, plus max|err| vs an fp32 torch forward on rank 0.

    python -m torch.distributed.run --nproc-per-node N tools/mlp_peer_bench.py [--tokens T]
"""
import argparse
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2302_02599_b200 import ShardingSpec  # noqa: E402
from paper_2302_02599_b200.runtime import MatmulStrategy, PeerMesh  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=16384)
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    ws, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    dev = int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")
    M, D, H = args.tokens, 1024, 4096
    g = torch.Generator(device="cuda").manual_seed(2302)
    x = torch.randn(M, D, device="cuda", generator=g).bfloat16()
    w1 = (torch.randn(D, H, device="cuda", generator=g) / 32).bfloat16()
    w2 = (torch.randn(H, D, device="cuda", generator=g) / 64).bfloat16()
    hs = H // ws
    w1s = w1[:, rank * hs:(rank + 1) * hs].contiguous()   # RS0 [D, H/ws]
    w2s = w2[rank * hs:(rank + 1) * hs].contiguous()      # S0R [H/ws, D]
    p = lambda s: ShardingSpec.parse(s, 1)  # noqa: E731
    fc1 = MatmulStrategy("split-n:0", p("RR"), p("RS0"), p("RS0"))
    fc2 = MatmulStrategy("split-k:0", p("RS0"), p("S0R"), p("RR"), [0])
    pm = PeerMesh([ws], rank, dev, 16)
    stream = torch.cuda.current_stream()

    def forward():
        h = pm.sharded_matmul(fc1, x, w1s, gelu=True, stream=stream)
        return pm.sharded_matmul(fc2, h, w2s, stream=stream)

    y = forward()
    torch.cuda.synchronize()
    err = None
    if rank == 0:
        ref = torch.nn.functional.gelu(x.float() @ w1.float()) @ w2.float()
        err = ((y.double() - ref.double()).abs().max() / ref.abs().max()).item()
    for _ in range(3):
        forward()
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(args.iters):
        forward()
    b.record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) / args.iters], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t[0])
    flops = 2 * 2.0 * M * D * H
    if rank == 0:
        print(json.dumps({"config": "configs[4]: GPT-2-medium MLP, Megatron split-n:0 / split-k:0",
                          "n_gpus": ws, "tokens": M, "transport": "peer (fused GEMM + all-reduce)",
                          "ms_per_forward": round(ms, 4),
                          "tflops_job": round(flops / ms / 1e9, 1), "max_rel_err": err}),
              flush=True)
    dist.barrier()
    pm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
