"""The reference's own layout tests (proj/tests/test_layout.cpp), re-expressed
against the drop-in API (C++ autoplan through libapl.so)."""
import itertools
import random

import pytest

from paper_2302_02599_b200 import (AxisError, CollectiveKind, DeviceMesh, DimSpec,
                                   PathCache, RankMismatchError, SchemaError, ShapeError,
                                   ShardingSpec, TensorMeta, conversion_cost, dim_diff,
                                   find_transform_path, heuristic_diff, one_step_transforms,
                                   parse_mesh_shape, collective_cost)

SQUARE = TensorMeta((8, 8), 4)


def mesh24():
    return DeviceMesh.uniform([2, 4])


def names(ts):
    return {str(s) for s, _ in ts}


def all_valid_specs(meta, mesh):
    """Independent enumeration (reference tests/helpers.hpp:245-276)."""
    rank, mr = len(meta.shape), mesh.rank()
    out = []

    def rec(d, used, dims):
        if d == rank:
            s = ShardingSpec(tuple(DimSpec(tuple(a)) for a in dims), mr)
            if s.valid_for(meta, mesh):
                out.append(s)
            return
        rec(d + 1, used, dims + [[]])

        def ext(cur, used):
            for a in range(mr):
                if a in used:
                    continue
                nxt = cur + [a]
                rec(d + 1, used | {a}, dims + [nxt])
                ext(nxt, used | {a})

        ext([], used)

    rec(0, frozenset(), [])
    return out


def apply_step(step, spec):
    """Reference tests/helpers.hpp:282-311."""
    dims = [list(d.axes) for d in spec.dims]
    d = dims[step.tensor_dim]
    if step.kind == CollectiveKind.kAllGather:
        assert d and d[-1] == step.mesh_axis
        d.pop()
    elif step.kind == CollectiveKind.kShardSlice:
        assert step.mesh_axis not in spec.used_axes()
        d.append(step.mesh_axis)
    elif step.kind == CollectiveKind.kAllToAll:
        assert step.target_dim != step.tensor_dim and d and d[-1] == step.mesh_axis
        d.pop()
        dims[step.target_dim].append(step.mesh_axis)
    else:
        raise AssertionError("reduce kinds never appear in paths")
    return ShardingSpec(tuple(DimSpec(tuple(a)) for a in dims), spec.mesh_rank)


def replay_ok(path, mesh, meta):
    cur = path.source
    for s in path.steps:
        cur = apply_step(s, cur)
        assert cur == s.result
        assert cur.valid_for(meta, mesh)
    return cur == path.target


def bfs(src, tgt, mesh, meta):
    if src == tgt:
        return 0
    seen, frontier = {str(src)}, [(src, 0)]
    for spec, depth in frontier:
        for nxt, _ in one_step_transforms(spec, mesh, meta):
            if nxt == tgt:
                return depth + 1
            if str(nxt) not in seen:
                seen.add(str(nxt))
                frontier.append((nxt, depth + 1))
    return -1


def test_spec_text_round_trips():
    assert str(ShardingSpec.parse("S0R", 2)) == "S0R"
    assert str(ShardingSpec.parse("RR", 2)) == "RR"
    assert str(ShardingSpec.parse("S01S2", 3)) == "S01S2"
    assert str(ShardingSpec.replicated(2, 2)) == "RR"
    assert str(ShardingSpec.parse("S10R", 2)) == "S10R"
    assert ShardingSpec.parse("S0R", 2) == ShardingSpec((DimSpec((0,)), DimSpec()), 2)
    with pytest.raises(AxisError):
        ShardingSpec.parse("S9R", 2)
    with pytest.raises(AxisError):
        ShardingSpec.parse("S0S0", 2)
    with pytest.raises(SchemaError):
        ShardingSpec.parse("XZ", 2)
    with pytest.raises(SchemaError):
        ShardingSpec.parse("SR", 2)
    with pytest.raises(SchemaError):
        ShardingSpec.parse("", 2)


def test_validity_axis_uniqueness_and_divisibility():
    m = mesh24()
    assert ShardingSpec.parse("S0S1", 2).valid_for(SQUARE, m)
    assert ShardingSpec.parse("S01R", 2).valid_for(SQUARE, m)
    assert not ShardingSpec((DimSpec((0,)), DimSpec((0,))), 2).valid_for(SQUARE, m)
    odd = TensorMeta((3, 8), 4)
    assert not ShardingSpec.parse("S0R", 2).valid_for(odd, m)
    assert ShardingSpec.parse("RS1", 2).valid_for(odd, m)
    assert not ShardingSpec((DimSpec((5,)), DimSpec()), 2).valid_for(SQUARE, m)


def test_per_device_bytes():
    m = DeviceMesh.uniform([4, 2])
    big = TensorMeta((1024, 1024), 4)
    assert ShardingSpec.replicated(2, 2).per_device_bytes(big, m) == 1024 * 1024 * 4
    assert ShardingSpec.parse("S0R", 2).per_device_bytes(big, m) == 1024 * 1024
    assert ShardingSpec.parse("S01R", 2).per_device_bytes(big, m) == 1024 * 1024 // 2
    assert ShardingSpec.parse("S0S1", 2).shard_count(m) == 8


def test_one_step_sets():
    assert names(one_step_transforms(ShardingSpec.parse("S0R", 2), mesh24(), SQUARE)) == \
        {"RR", "S0S1", "S01R", "RS0"}
    ts = one_step_transforms(ShardingSpec.replicated(2, 2), mesh24(), SQUARE)
    assert names(ts) == {"S0R", "S1R", "RS0", "RS1"}
    assert all(s.kind == CollectiveKind.kShardSlice for _, s in ts)
    odd = TensorMeta((3, 8), 4)
    assert names(one_step_transforms(ShardingSpec.replicated(2, 2), mesh24(), odd)) == \
        {"RS0", "RS1"}


def test_dim_and_heuristic_diff():
    r, s0, s1 = DimSpec(), DimSpec((0,)), DimSpec((1,))
    assert dim_diff(r, r) == 0
    assert dim_diff(s0, s0) == 0
    assert dim_diff(s0, s1) == 5
    assert dim_diff(s0, r) == 2
    assert dim_diff(r, s0) == 1
    s0r, rs0 = ShardingSpec.parse("S0R", 2), ShardingSpec.parse("RS0", 2)
    assert heuristic_diff(s0r, s0r) == 0
    assert heuristic_diff(s0r, rs0) == 3
    assert heuristic_diff(ShardingSpec.parse("S0S1", 2), ShardingSpec.replicated(2, 2)) == 4
    with pytest.raises(RankMismatchError):
        heuristic_diff(s0r, ShardingSpec.replicated(3, 2))
    specs = all_valid_specs(SQUARE, mesh24())
    for a, b in itertools.product(specs, specs):
        assert (heuristic_diff(a, b) == 0) == (a == b)


def test_full_rank2_enumeration_replays_within_bfs_plus_two():
    """Acceptance criterion 1 (acceptance_test.cpp:124-163)."""
    m = mesh24()
    specs = all_valid_specs(SQUARE, m)
    assert len(specs) == 11
    for src, tgt in itertools.product(specs, specs):
        p = find_transform_path(src, tgt, m, SQUARE)
        assert replay_ok(p, m, SQUARE), (str(src), str(tgt))
        opt = bfs(src, tgt, m, SQUARE)
        assert 0 <= opt and len(p.steps) <= opt + 2
        if src == tgt:
            assert not p.steps


def test_published_paths():
    m = mesh24()
    p = find_transform_path(ShardingSpec.parse("S0R", 2), ShardingSpec.parse("S0R", 2), m, SQUARE)
    assert not p.steps and conversion_cost(p, m, SQUARE) == 0.0
    p = find_transform_path(ShardingSpec.parse("S0R", 2), ShardingSpec.parse("RS0", 2), m, SQUARE)
    assert len(p.steps) == 1
    s = p.steps[0]
    assert (s.kind, s.tensor_dim, s.target_dim, s.mesh_axis) == (CollectiveKind.kAllToAll, 0, 1, 0)
    p = find_transform_path(ShardingSpec.parse("S01R", 2), ShardingSpec.replicated(2, 2), m,
                            SQUARE)
    assert [(x.kind, x.mesh_axis) for x in p.steps] == [(CollectiveKind.kAllGather, 1),
                                                        (CollectiveKind.kAllGather, 0)]


def test_conversion_cost():
    m = DeviceMesh.uniform([4])
    big = TensorMeta((1024, 1024), 4)
    p = find_transform_path(ShardingSpec.parse("S0R", 1), ShardingSpec.replicated(2, 1), m, big)
    assert len(p.steps) == 1
    expected = 3e-5 + 0.75 * 1048576 * 1e-9
    assert abs(conversion_cost(p, m, big) - expected) <= 1e-12 * expected
    assert abs(p.comm_cost_s - expected) <= 1e-12 * expected
    m2 = mesh24()
    p = find_transform_path(ShardingSpec.parse("S01R", 2), ShardingSpec.replicated(2, 2), m2,
                            SQUARE)
    total = p.comm_cost_s
    hop_sum, cur = 0.0, p.source
    for s in p.steps:
        hop_sum += collective_cost(m2, [s.mesh_axis], s.kind, cur.per_device_bytes(SQUARE, m2))
        cur = s.result
    assert abs(total - hop_sum) <= 1e-12 * total


def test_ring_formulas():
    """Reference test_cluster.cpp:140-210 pricing pins."""
    m = DeviceMesh.uniform([4])
    ar = collective_cost(m, [0], CollectiveKind.kAllReduce, 1 << 20)
    ag = collective_cost(m, [0], CollectiveKind.kAllGather, 1 << 20)
    rs = collective_cost(m, [0], CollectiveKind.kReduceScatter, 1 << 20)
    assert ag == rs
    assert abs(ar - (ag + rs)) < 1e-18
    assert collective_cost(m, [0], CollectiveKind.kShardSlice, 1 << 20) == 0.0
    with pytest.raises(AxisError):
        collective_cost(m, [3], CollectiveKind.kAllGather, 10)


def test_path_cache():
    m = mesh24()
    cache = PathCache()
    src, tgt = ShardingSpec.parse("S0R", 2), ShardingSpec.parse("RS0", 2)
    first = cache.get(src, tgt, m, SQUARE)
    assert cache.searches() == 1
    second = cache.get(src, tgt, m, SQUARE)
    assert cache.searches() == 1
    assert second.comm_cost_s == first.comm_cost_s and len(second.steps) == len(first.steps)
    cache.get(src, tgt, m, TensorMeta((16, 8), 4))
    assert cache.searches() == 2
    cache.get(src, tgt, DeviceMesh.uniform([4, 2]), SQUARE)
    assert cache.searches() == 3 and cache.size() == 3
    cache.clear()
    assert cache.size() == 0
    assert cache.get(src, tgt, m, SQUARE).comm_cost_s == first.comm_cost_s


def test_random_rank3_pairs_are_sound():
    m = DeviceMesh.uniform([2, 2, 2])
    meta = TensorMeta((8, 4, 2), 4)
    specs = all_valid_specs(meta, m)
    assert len(specs) > 10
    rng = random.Random(271828)
    for _ in range(200):
        a, b = rng.choice(specs), rng.choice(specs)
        assert replay_ok(find_transform_path(a, b, m, meta), m, meta)


def test_invalid_endpoints_raise_shape_error():
    m = mesh24()
    with pytest.raises(ShapeError):
        find_transform_path(ShardingSpec.parse("S0R", 2), ShardingSpec.parse("S01R", 2), m,
                            TensorMeta((4, 8), 4))


def test_mesh_shape_parse():
    assert parse_mesh_shape("2x4") == (2, 4)
    assert parse_mesh_shape("8") == (8,)
    for bad in ["2x", "x2", "", "2xx4", "0x2", "axb"]:
        with pytest.raises(SchemaError):
            parse_mesh_shape(bad)
