"""Sharded-matmul strategy catalog == the reference's generate_strategies
(golden from oracle/_ref: tests/golden/strategies.json), entry for entry:
names, order, specs, partial-sum axes and the priced times/bytes."""
import json
from pathlib import Path

import pytest

from paper_2302_02599_b200 import DeviceMesh, TensorMeta
from paper_2302_02599_b200.strategies import matmul_strategies

GOLDEN = json.loads((Path(__file__).resolve().parent / "golden" / "strategies.json").read_text())


def operand_metas(graph, node_id):
    nodes = {n["id"]: n for n in graph["nodes"]}
    node = nodes[node_id]
    metas = []
    shapes = {}
    for n in graph["nodes"]:  # infer matmul output shapes in order
        if n["outputs"]:
            shapes[n["id"]] = tuple(n["outputs"][0]["shape"])
        elif n["kind"] in ("matmul", "batched-matmul"):
            a, b = shapes[n["inputs"][0][0]], shapes[n["inputs"][1][0]]
            shapes[n["id"]] = a[:-1] + (b[-1],)
        elif n["kind"] in ("elementwise-unary",):
            shapes[n["id"]] = shapes[n["inputs"][0][0]]
    for ref, _ in node["inputs"]:
        metas.append(TensorMeta(shapes[ref], 2))
    return metas


@pytest.mark.parametrize("case", GOLDEN["cases"],
                         ids=[f"{c['node']}-{'x'.join(map(str, c['mesh']))}" for c in GOLDEN["cases"]])
def test_catalog_matches_reference(case):
    graph = GOLDEN["graphs"][case["graph"]]
    a, b = operand_metas(graph, case["node"])
    mesh = DeviceMesh.uniform(case["mesh"], device_flops_per_s=case["flops"])
    mine = matmul_strategies(mesh, a, b, batched=case["graph"] == "bmm")
    want = case["strategies"]
    assert [s.name for s in mine] == [w["name"] for w in want]
    for s, w in zip(mine, want):
        assert (str(s.a), str(s.b), str(s.c)) == (w["a"], w["b"], w["c"]), w["name"]
        assert s.partial_sum == w["partial_sum"] and list(s.reduce_axes) == w["reduce_axes"]
        assert repr(s.compute_time_s) == repr(float(w["compute_time_s"])), w["name"]
        assert repr(s.comm_time_s) == repr(float(w["comm_time_s"])), w["name"]
        assert s.memory_bytes == w["memory_bytes"]


def test_survey_candidate_counts():
    """fc1/fc2 have 4 on [8], 16 on 2x4, 37 on 2x2x2."""
    x, w1 = TensorMeta((16384, 1024), 2), TensorMeta((1024, 4096), 2)
    assert len(matmul_strategies(DeviceMesh.uniform([8]), x, w1)) == 4
    assert len(matmul_strategies(DeviceMesh.uniform([2, 4]), x, w1)) == 16
    assert len(matmul_strategies(DeviceMesh.uniform([2, 2, 2]), x, w1)) == 37
