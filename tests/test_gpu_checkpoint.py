"""Activation checkpointing as the plan schedules it (reference ckpt.cpp:
Rotor over the chain stages; plan["schedule"] decides store_all /
store_boundary / recompute per stage and groups the non-store_all runs into
recompute blocks, plan_to_json planner.cpp:455-600). The reference planner's
own plans under a tight budget (tests/golden/make_plans.py: the GPT-2 MLP at
88 MiB on [8] and [2,4] checkpoints fc1+gelu; the GPT block at 100 MiB on [8]
checkpoints the whole attention stage) run with the schedule honoured:

* after the forward pass the checkpointed stages hold no backward state and
  fewer bytes stay resident than with everything stored;
* backward re-runs each block once, from its boundary values, and every
  gradient is byte-identical to the store-everything run (the recompute is
  the same kernels on the same bytes)."""
import json
from pathlib import Path

import pytest
import torch

from paper_2302_02599_b200.executor import PlanExecutor
from paper_2302_02599_b200.runtime import Mesh

pytestmark = pytest.mark.gpu
PLANS = Path(__file__).resolve().parent / "golden" / "plans"
CKPT_PLANS = ["gpt2_mlp_mesh8_88.json", "gpt2_mlp_mesh2x4_88.json",
              "gpt_block_b4s1024_mesh8_100.json"]


def _mlp_case():
    graph = json.loads((PLANS / "gpt2_mlp_graph.json").read_text())
    g = torch.Generator(device="cuda").manual_seed(5)
    feeds = {"x": torch.randn(16384, 1024, device="cuda", generator=g).bfloat16(),
             "w1": (torch.randn(1024, 4096, device="cuda", generator=g) / 32).bfloat16(),
             "w2": (torch.randn(4096, 1024, device="cuda", generator=g) / 64).bfloat16()}
    return graph, feeds


def _case(name):
    if name.startswith("gpt2_mlp"):
        return _mlp_case()
    import sys
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from test_gpu_block import _case as block_case

    graph, feeds, _ = block_case("b4s1024")
    return graph, feeds


def _step(graph, plan, feeds, checkpoint):
    ex = PlanExecutor(Mesh.local(plan["mesh"]["shape"]), graph, plan, checkpoint=checkpoint)
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    outs = ex.forward(feeds, train=True)
    torch.cuda.synchronize()
    resident = torch.cuda.memory_allocated() - base
    torch.manual_seed(3)
    gy = torch.randn(outs[0].shape, device="cuda").bfloat16()
    grads = ex.backward(gy)
    torch.cuda.synchronize()
    return ex, outs, grads, resident


@pytest.mark.parametrize("name", CKPT_PLANS)
def test_checkpoint_schedule_recomputes_with_identical_gradients(cuda, name):
    plan = json.loads((PLANS / name).read_text())
    sched = plan["schedule"]
    assert any(d != "store_all" for d in sched["decision"])  # the fixture checkpoints
    graph, feeds = _case(name)

    ex, outs, grads, resident = _step(graph, plan, feeds, checkpoint=True)
    blocks = {b for b in sched["block_index"] if b >= 0}
    assert set(ex._blocks) == blocks and ex._recomputed == blocks
    members = {m for ms in ex._blocks.values() for m in ms}
    assert members and all(
        m in {s for st in plan["stages"] if sched["block_index"][st["index"]] >= 0
              for s in st["members"]} for m in members)
    del ex

    ex0, outs0, grads0, resident0 = _step(graph, plan, feeds, checkpoint=False)
    assert not ex0._blocks
    assert resident < resident0, (resident, resident0)
    for a, b in zip(outs, outs0):
        assert torch.equal(a, b)
    assert grads.keys() == grads0.keys() and grads
    for k in grads:
        for a, b in zip(grads[k], grads0[k]):
            assert torch.equal(a, b), k
