"""The transformer block (gpt_block, GPT-2-medium width) executed distributed
over peer memory: 8 processes, one per mesh device, sharing cuda:0 through
CUDA IPC (on an 8-GPU box the same code reads over NVLink), run the
reference planner's b8s1024 plans ([8], 2x4, 2x2x2) with the PlanExecutor on
a PeerRuntime -- conversions as pull kernels, the embedding table read from
its owners' blocks over peer memory, partial sums (layernorm / embedding /
batched-matmul gradients) as in-place peer all-reduces. Every rank's
forward output and its shard of every parameter gradient against fp32 torch
autograd on the same bf16 operands (tolerances of test_gpu_block.py)."""
import json
import os
import socket
import sys
from pathlib import Path

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

HERE = Path(__file__).resolve().parent
PLANS = HERE / "golden" / "plans"
NAMES = ["gpt_block_b8s1024_mesh8_unlimited.json", "gpt_block_b8s1024_mesh2x4_unlimited.json",
         "gpt_block_b8s1024_mesh2x2x2_unlimited.json"]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    sys.path.insert(0, str(HERE))
    from test_gpu_block import PARAMS, _operands, block_reference
    from test_gpu_peer_executor import _shard

    from paper_2302_02599_b200.executor import PlanExecutor
    from paper_2302_02599_b200.peer import PeerRuntime

    graph = json.loads((PLANS / "gpt_block_b8s1024_graph.json").read_text())
    try:
        feeds = _operands(graph)
        leaves = {k: feeds[k].float().requires_grad_() for k in PARAMS}
        p = dict(feeds)
        p.update(leaves)
        ref_out = block_reference(p)
        torch.manual_seed(7)
        gy = torch.randn(ref_out.shape, device="cuda").bfloat16()
        ref_out.backward(gy.float())
        ref_out = ref_out.detach()
        ref = {k: v.grad for k, v in leaves.items()}
        del leaves, p
        for name in NAMES:
            plan = json.loads((PLANS / name).read_text())
            rt = PeerRuntime(plan["mesh"]["shape"], rank, 0, heap_bytes=3 << 30)
            ex = PlanExecutor(rt, graph, plan)
            out = ex.forward(feeds)[0]
            torch.cuda.synchronize()
            err = ((out.float() - ref_out).abs().max() / ref_out.abs().max()).item()
            ok = err <= 4e-2
            for _ in range(2):  # the second step recycles the heap
                ex.forward(feeds, train=True)
                grads = ex.backward(gy)
            torch.cuda.synchronize()
            for k in PARAMS:
                want = _shard(ref[k], ex.spec[k], rt.geo, rank)
                g = grads[k][0].float()
                mx = ((g - want).abs().max() / want.abs().max()).item()
                mean = ((g - want).abs().mean() / want.abs().mean()).item()
                ok = ok and g.shape == want.shape and mx <= 2e-2 and mean <= 1.5e-2
                err = max(err, mx)
            q.put((rank, name, ok, err))
            torch.cuda.synchronize()
            dist.barrier()
            rt.close()
            dist.barrier()
    finally:
        dist.destroy_process_group()


def test_block_plans_over_peer_memory(cuda):
    world = 8
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=900)
    res = []
    while not q.empty():
        res.append(q.get())
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert len(res) == world * len(NAMES), res
    assert all(r[2] for r in res), [r for r in res if not r[2]]
