"""BASELINE config 5 on N GPUs over peer memory (one process per GPU): the
GPT-2-medium MLP executed by the PlanExecutor on a PeerRuntime -- the pinned
Megatron plan (fc1 split-n:0 local GEMM + GELU; fc2 split-k:0 GEMM +
all-reduce fused over peer memory) or a reference planner plan
(conversions as one pull kernel per rank, partial sums as one peer
all-reduce kernel). Prints one JSON line (rank 0): ms per forward and per
training step (max over ranks), TFLOP/s of the whole job, and the max
relative error of the forward vs an fp32 torch forward.

    python -m torch.distributed.run --nproc-per-node N tools/mlp_peer_bench.py \\
        [--plan megatron|tests/golden/plans/gpt2_mlp_mesh2x4_unlimited.json]
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

from paper_2302_02599_b200.executor import PlanExecutor, megatron_mlp_plan  # noqa: E402
from paper_2302_02599_b200.peer import PeerRuntime  # noqa: E402

GRAPH = json.loads((ROOT / "tests" / "golden" / "plans" / "gpt2_mlp_graph.json").read_text())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--plan", default="megatron")
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    ws, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    dev = int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")
    plan = megatron_mlp_plan() if args.plan == "megatron" else json.loads(Path(args.plan).read_text())
    shape = plan["mesh"]["shape"] if "mesh" in plan else [ws]
    g = torch.Generator(device="cuda").manual_seed(2302)
    x = torch.randn(16384, 1024, device="cuda", generator=g).bfloat16()
    w1 = (torch.randn(1024, 4096, device="cuda", generator=g) / 32).bfloat16()
    w2 = (torch.randn(4096, 1024, device="cuda", generator=g) / 64).bfloat16()
    gy = torch.randn(16384, 1024, device="cuda", generator=g).bfloat16()
    rt = PeerRuntime(shape, rank, dev, heap_bytes=2 << 30)
    ex = PlanExecutor(rt, GRAPH, plan)
    shards = {k: ex.shard(k, v) for k, v in {"x": x, "w1": w1, "w2": w2}.items()}
    stream = torch.cuda.current_stream()
    y = ex.forward(shards, stream=stream)[0]
    torch.cuda.synchronize()
    ref = torch.nn.functional.gelu(x.float() @ w1.float()) @ w2.float()
    err = ((y.double() - ref.double()).abs().max() / ref.abs().max()).item()

    def time_it(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.iters):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b) / args.iters], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t[0])

    fwd = time_it(lambda: ex.forward(shards, stream=stream))

    def train():
        ex.forward(shards, stream=stream, train=True)
        ex.backward(gy, stream=stream)

    trn = time_it(train)
    flops = 2 * 2.0 * 16384 * 1024 * 4096
    if rank == 0:
        print(json.dumps({"config": "configs[4]: GPT-2-medium MLP", "plan": args.plan,
                          "mesh": shape, "n_gpus": ws, "transport": "peer (PeerRuntime)",
                          "strategies": {k: v.name for k, v in ex.strategy.items()},
                          "ms_per_forward": round(fwd, 4),
                          "tflops_forward_job": round(flops / fwd / 1e9, 1),
                          "ms_per_train_step": round(trn, 4),
                          "tflops_train_job": round(2.5 * flops / trn / 1e9, 1),
                          "max_rel_err": err}), flush=True)
    torch.cuda.synchronize()
    dist.barrier()
    rt.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
