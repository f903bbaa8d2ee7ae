"""The plan's checkpoint schedule on a distributed mesh: 8 processes on cuda:0
over the NCCL transport (one NCCL_HOSTID per rank, as in test_gpu_nccl.py),
running the reference planner's checkpointing MLP plans
(gpt2_mlp_mesh8_88 / gpt2_mlp_mesh2x4_88: fc1 + gelu recomputed, Rotor
schedule from ckpt.cpp). On every rank the recompute block runs once in
backward (its weight all-gather re-issued over NCCL) and every local
gradient shard is byte-identical to the same rank's store-everything run."""
import json
import os
from pathlib import Path

import pytest
import torch.multiprocessing as mp

from test_gpu_nccl import _port, drain

pytestmark = pytest.mark.gpu
PLANS = Path(__file__).resolve().parent / "golden" / "plans"


def _worker(rank, world, port, names, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                      NCCL_HOSTID=f"apl-ckpt-test-host-{rank}", NCCL_SOCKET_IFNAME="lo",
                      NCCL_IB_DISABLE="1")
    import torch
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2302_02599_b200.executor import PlanExecutor
    from paper_2302_02599_b200.runtime import Mesh

    graph = json.loads((PLANS / "gpt2_mlp_graph.json").read_text())
    g = torch.Generator(device="cuda").manual_seed(5)
    feeds = {"x": torch.randn(16384, 1024, device="cuda", generator=g).bfloat16(),
             "w1": (torch.randn(1024, 4096, device="cuda", generator=g) / 32).bfloat16(),
             "w2": (torch.randn(4096, 1024, device="cuda", generator=g) / 64).bfloat16()}
    gy = torch.randn(16384, 1024, device="cuda", generator=g).bfloat16()
    try:
        for name in names:
            plan = json.loads((PLANS / name).read_text())
            mesh = Mesh.from_process_group(plan["mesh"]["shape"])
            stream = torch.cuda.current_stream()
            runs = {}
            for ckpt in (True, False):
                ex = PlanExecutor(mesh, graph, plan, checkpoint=ckpt)
                outs = ex.forward(feeds, stream=stream, train=True)
                grads = ex.backward(gy, stream=stream)
                mesh.synchronize(stream, timeout_s=300)
                runs[ckpt] = ({k: [t.clone() for t in v] for k, v in grads.items()},
                              outs[0].clone(), set(getattr(ex, "_recomputed", set())),
                              set(ex._blocks))
            (g1, o1, rec, blocks), (g0, o0, rec0, blocks0) = runs[True], runs[False]
            same = (g1.keys() == g0.keys() and bool(g1) and torch.equal(o1, o0) and
                    all(torch.equal(a, b) for k in g1 for a, b in zip(g1[k], g0[k])))
            q.put((name, rank, bool(blocks) and rec == blocks and not blocks0, same,
                   sorted(g1)))
            dist.barrier()
            mesh.close()
    finally:
        dist.destroy_process_group()


def test_checkpoint_schedule_over_nccl(cuda):
    names = ["gpt2_mlp_mesh8_88.json", "gpt2_mlp_mesh2x4_88.json"]
    world = 8
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, names, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = drain(procs, q, 1200)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert len(res) == world * len(names), res
    for name, rank, recomputed, same, keys in res:
        assert recomputed, (name, rank)
        assert same, (name, rank)
        assert set(keys) == {"w1", "w2"}, keys
