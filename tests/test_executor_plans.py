"""Plan ingestion (CPU): the executor decodes every committed reference plan
(tests/golden/plans, written by the reference planner via oracle/_ref) and
the communication it would issue equals the plan's inserted_comm_nodes
(reference planner.cpp:218-352) step for step."""
import json
from pathlib import Path

import pytest

from paper_2302_02599_b200 import DeviceMesh
from paper_2302_02599_b200.executor import PlanExecutor, megatron_mlp_plan

PLANS = Path(__file__).resolve().parent / "golden" / "plans"
GRAPH = json.loads((PLANS / "gpt2_mlp_graph.json").read_text())


class _GeoOnly:
    """Host-only stand-in for runtime.Mesh (geometry, no device)."""

    def __init__(self, shape):
        self.geo = DeviceMesh.uniform(shape)
        self.num_devices = self.geo.num_devices()
        self.num_local = self.num_devices
        self.distributed = False
        self.first_local = 0


@pytest.mark.parametrize("path", sorted(p.name for p in PLANS.glob("gpt2_mlp_mesh*.json")))
def test_reference_plans_decode_and_match_communication(path):
    plan = json.loads((PLANS / path).read_text())
    ex = PlanExecutor(_GeoOnly(plan["mesh"]["shape"]), GRAPH, plan)
    ex.check_against_plan()
    assert ex.strategy["fc1"].name == plan["nodes"]["fc1"]["strategy"]


def test_megatron_plan_decodes():
    ex = PlanExecutor(_GeoOnly([8]), GRAPH, megatron_mlp_plan())
    ex.check_against_plan()
    assert ex.strategy["fc1"].name == "split-n:0" and ex.strategy["fc2"].partial_sum
    assert ex._fusable_gelu("fc1") == "gelu"


@pytest.mark.parametrize("path", sorted(p.name for p in PLANS.glob("gpt_block_*_mesh*.json")))
def test_block_plans_decode_and_match_communication(path):
    """The reference's transformer-block plans (embedding, layernorm, reshape,
    transpose, batched matmul, softmax, elementwise strategies): every
    non-matmul strategy decodes to input layouts whose conversions are
    exactly the plan's inserted communication."""
    tag = path.split("_mesh")[0]
    graph = json.loads((PLANS / f"{tag}_graph.json").read_text())
    plan = json.loads((PLANS / path).read_text())
    ex = PlanExecutor(_GeoOnly(plan["mesh"]["shape"]), graph, plan)
    ex.check_against_plan()
    assert ex.unary_op("mask2") == ("not",)
    assert ex.unary_op("act") == ("gelu",)
    op, alpha = ex.unary_op("scaled")
    h = ex.shapes["qr"][0][-1]
    assert op == "scale" and abs(alpha - h ** -0.5) < 1e-12
    assert ex.strategy["scores"].name == plan["nodes"]["scores"]["strategy"]
    # reshape strategies: the plan's rewritten local target shape is the
    # local shape of the node's spec (a view of the producer's shard)
    for rw in plan.get("reshape_rewrites", []):
        nid = rw["node"]
        assert list(ex.spec[nid].local_shape(ex._meta(nid), ex.geo)) == rw["new_target_shape"]


def test_unnamed_unary_is_rejected_unless_bound():
    """The graph format does not name elementwise-unary functions; a unary
    node the executor cannot identify (here one renamed to hide the
    attention-scale role) is refused instead of silently becoming GELU, and
    an explicit unary= binding executes it."""
    graph = json.loads((PLANS / "gpt_block_fixture_graph.json").read_text())
    plan = json.loads((PLANS / "gpt_block_fixture_mesh4_unlimited.json").read_text())
    ren = {"scaled": "mystery"}
    for n in graph["nodes"]:
        n["id"] = ren.get(n["id"], n["id"])
        n["inputs"] = [[ren.get(a, a), i] for a, i in n["inputs"]]
    plan["nodes"] = {ren.get(k, k): v for k, v in plan["nodes"].items()}
    for c in plan.get("inserted_comm_nodes", []):
        for key in ("producer", "consumer"):
            if c.get(key) in ren:
                c[key] = ren[c[key]]
    with pytest.raises(ValueError, match="mystery"):  # rejected up front
        PlanExecutor(_GeoOnly(plan["mesh"]["shape"]), graph, plan)
    ex2 = PlanExecutor(_GeoOnly(plan["mesh"]["shape"]), graph, plan,
                       unary={"mystery": ("scale", 0.125)})
    assert ex2.unary_op("mystery") == ("scale", 0.125)


@pytest.mark.parametrize("path", ["gpt2_mlp_mesh8_88.json", "gpt2_mlp_mesh2x4_88.json",
                                  "gpt_block_b4s1024_mesh8_100.json"])
def test_checkpoint_blocks_follow_the_schedule(path):
    """Recompute blocks (executor._checkpoint_blocks) are exactly the stages
    the reference schedule marks with a block index (ckpt.cpp decisions
    store_boundary / recompute), members in graph order; checkpoint=False
    (or a store_all schedule) has none."""
    plan = json.loads((PLANS / path).read_text())
    tag = path.split("_mesh")[0]
    graph = GRAPH if tag == "gpt2_mlp" else json.loads((PLANS / f"{tag}_graph.json").read_text())
    ex = PlanExecutor(_GeoOnly(plan["mesh"]["shape"]), graph, plan)
    sched = plan["schedule"]
    want = {}
    for st in plan["stages"]:
        b = sched["block_index"][st["index"]]
        if b >= 0:
            want.setdefault(b, set()).update(st["members"])
    assert want and {b: set(m) for b, m in ex._blocks.items()} == want
    order = [n["id"] for n in graph["nodes"]]
    for ms in ex._blocks.values():
        assert ms == sorted(ms, key=order.index)
    if tag == "gpt2_mlp":
        assert set(ex._blocks[0]) == {"fc1", "gelu"}
        assert ex._fusable_gelu("fc1") == "gelu"  # same block: still fused
    assert not PlanExecutor(_GeoOnly(plan["mesh"]["shape"]), graph, plan,
                            checkpoint=False)._blocks
    store_all = json.loads((PLANS / "gpt2_mlp_mesh8_unlimited.json").read_text())
    assert not PlanExecutor(_GeoOnly([8]), GRAPH, store_all)._blocks


def test_checkpoint_off_on_bump_allocator_meshes():
    """A mesh with its own per-step allocator (the peer runtime's symmetric
    heap) frees nothing mid-step, so the executor stores everything there."""
    plan = json.loads((PLANS / "gpt2_mlp_mesh8_88.json").read_text())

    class _HeapMesh(_GeoOnly):
        def empty(self, shape, dtype):  # pragma: no cover - never called here
            raise AssertionError

    assert PlanExecutor(_GeoOnly([8]), GRAPH, plan)._blocks
    assert not PlanExecutor(_HeapMesh([8]), GRAPH, plan)._blocks
