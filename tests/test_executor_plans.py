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
