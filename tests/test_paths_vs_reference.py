"""Drop-in parity: every path the C++ host API produces equals the
reference's, step for step and bit-for-bit in cost.

Pinned two ways:
  * committed golden paths from the reference library (tests/golden/,
    written by tests/golden/make_golden.py from oracle/_ref) — runs anywhere;
  * live against oracle/_ref (the reference compiled from /root/reference)
    on extra random cases, when that library is present.
"""
import gzip
import json
import random
from pathlib import Path

import pytest

from paper_2302_02599_b200 import (DeviceMesh, ShardingSpec, TensorMeta, collective_cost,
                                   CollectiveKind, one_step_transforms, find_transform_path,
                                   PathCache)

GOLDEN = Path(__file__).resolve().parent / "golden"


def golden_cases():
    with gzip.open(GOLDEN / "paths.json.gz", "rt") as f:
        return json.load(f)["cases"]


CASES = golden_cases()


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_paths_match_reference_golden(case):
    mesh = DeviceMesh.uniform(case["mesh"])
    mr = len(case["mesh"])
    meta = TensorMeta(tuple(case["shape"]), case["dtype_bytes"])
    cache = PathCache()
    for src, tgt, steps, cost, bfs in case["pairs"]:
        s, t = ShardingSpec.parse(src, mr), ShardingSpec.parse(tgt, mr)
        p = find_transform_path(s, t, mesh, meta)
        got = [[int(x.kind), x.tensor_dim, x.target_dim, x.mesh_axis, str(x.result)]
               for x in p.steps]
        assert got == steps, (src, tgt)
        assert repr(p.comm_cost_s) == cost, (src, tgt, p.comm_cost_s, cost)
        assert len(p.steps) <= bfs + 2
        c = cache.get(s, t, mesh, meta)
        assert repr(c.comm_cost_s) == cost


def test_spec_enumeration_matches_reference_golden():
    from test_layout_api import all_valid_specs

    for case in CASES:
        mesh = DeviceMesh.uniform(case["mesh"])
        meta = TensorMeta(tuple(case["shape"]), case["dtype_bytes"])
        assert [str(s) for s in all_valid_specs(meta, mesh)] == case["specs"], case["name"]


def test_one_step_sets_match_reference_golden():
    for c in json.loads((GOLDEN / "one_step.json").read_text()):
        mesh = DeviceMesh.uniform(c["mesh"])
        meta = TensorMeta(tuple(c["shape"]), c["dtype_bytes"])
        got = [[int(s.kind), s.tensor_dim, s.target_dim, s.mesh_axis, str(n)]
               for n, s in one_step_transforms(ShardingSpec.parse(c["spec"], len(c["mesh"])),
                                               mesh, meta)]
        assert got == c["neighbours"], c["spec"]


def test_collective_costs_match_reference_golden():
    for c in json.loads((GOLDEN / "costs.json").read_text()):
        v = collective_cost(DeviceMesh.uniform(c["mesh"]), c["axes"], CollectiveKind(c["kind"]),
                            c["bytes"])
        assert repr(v) == c["cost"], c


def _ref():
    try:
        from oracle import ref
    except ImportError:
        return None
    return ref if ref.available() else None


@pytest.mark.skipif(_ref() is None, reason="reference library (oracle/_ref) not built")
def test_paths_match_live_reference_random_meshes():
    ref = _ref()
    rng = random.Random(2302)
    meshes = [[2], [3], [8], [2, 2], [2, 3], [3, 2], [2, 4], [4, 2], [2, 2, 2], [1, 4],
              [2, 1, 2], [2, 2, 2, 2]]
    for _ in range(60):
        mesh_shape = rng.choice(meshes)
        rank = rng.choice([1, 2, 3, 4])
        shape = [rng.choice([1, 2, 4, 6, 8, 12, 16]) for _ in range(rank)]
        eb = rng.choice([1, 2, 4, 8])
        specs = ref.all_valid_specs(mesh_shape, shape, eb)
        mesh = DeviceMesh.uniform(mesh_shape)
        meta = TensorMeta(tuple(shape), eb)
        for _ in range(25):
            a, b = rng.choice(specs), rng.choice(specs)
            rc, steps, cost = ref.find_path(mesh_shape, shape, eb, a, b)
            assert rc == 0
            p = find_transform_path(ShardingSpec.parse(a, len(mesh_shape)),
                                    ShardingSpec.parse(b, len(mesh_shape)), mesh, meta)
            got = [(int(x.kind), x.tensor_dim, x.target_dim, x.mesh_axis, str(x.result))
                   for x in p.steps]
            assert got == [tuple(s) for s in steps], (mesh_shape, shape, a, b)
            assert p.comm_cost_s == cost


@pytest.mark.skipif(_ref() is None, reason="reference library (oracle/_ref) not built")
def test_error_classes_match_live_reference():
    ref = _ref()
    from paper_2302_02599_b200 import AxisError, SchemaError, ShapeError

    codes = {SchemaError: 1, AxisError: 2, ShapeError: 3}
    for src, tgt, shape in [("S9R", "RR", [8, 8]), ("XR", "RR", [8, 8]), ("S0R", "S01R", [4, 8]),
                            ("S00", "RR", [8, 8]), ("SR", "RR", [8, 8])]:
        rc, _, _ = ref.find_path([2, 4], shape, 4, src, tgt)
        try:
            find_transform_path(ShardingSpec.parse(src, 2), ShardingSpec.parse(tgt, 2),
                                DeviceMesh.uniform([2, 4]), TensorMeta(tuple(shape), 4))
            mine = 0
        except tuple(codes) as e:
            mine = codes[type(e)]
        assert mine == rc, (src, tgt)
