"""GPU parity: conversions executed by libapl.so kernels on a simulated mesh
(every mesh device a buffer on cuda:0) must equal the CPU oracle bytewise —
stepwise along the reference path, and collapsed into one exchange."""
import gzip
import json
import random
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import data as O
from paper_2302_02599_b200 import (DeviceMesh, ShardingSpec, TensorMeta, find_transform_path,
                                   CollectiveKind)
from paper_2302_02599_b200.runtime import Mesh, launch_count

pytestmark = pytest.mark.gpu

GOLDEN = Path(__file__).resolve().parent / "golden"
_TORCH = {1: torch.uint8, 2: torch.int16, 4: torch.int32, 8: torch.int64}
_NP = {1: np.uint8, 2: np.int16, 4: np.int32, 8: np.int64}


def _cases():
    with gzip.open(GOLDEN / "paths.json.gz", "rt") as f:
        return {c["name"]: c for c in json.load(f)["cases"]}


CASES = _cases()


def to_dev(arrs):
    return [torch.from_numpy(np.ascontiguousarray(a).view(_NP[a.itemsize])).cuda() for a in arrs]


def check_conversion(mesh_shape, shape, eb, src, tgt, fuse, g=None, stream=None):
    mesh = Mesh.local(mesh_shape)
    mr = len(mesh_shape)
    meta = TensorMeta(tuple(shape), eb)
    if g is None:
        g = O.fill_global(tuple(shape), eb)
    s, t = ShardingSpec.parse(src, mr), ShardingSpec.parse(tgt, mr)
    path = find_transform_path(s, t, mesh.geo, meta)
    ins = to_dev(O.shards(g, O.parse_spec(src, mr), mesh_shape))
    outs = [torch.full(t.local_shape(meta, mesh.geo), -1, dtype=_TORCH[eb], device="cuda")
            for _ in range(mesh.num_devices)]
    mesh.run_path(path, meta, ins, outs, fuse=fuse, stream=stream)
    torch.cuda.synchronize()
    want = O.shards(g, O.parse_spec(tgt, mr), mesh_shape)
    for d, (o, w) in enumerate(zip(outs, want)):
        got = o.cpu().numpy().tobytes()
        assert got == w.tobytes(), f"{src}->{tgt} fuse={fuse} device {d}"
    return path


@pytest.mark.parametrize("fuse", [False, True])
def test_config1_s0r_to_rs0_on_simulated_2x2(cuda, fuse):
    path = check_conversion([2, 2], (1024, 1024), 4, "S0R", "RS0", fuse)
    assert [(int(s.kind), s.tensor_dim, s.target_dim, s.mesh_axis) for s in path.steps] == \
        [(int(CollectiveKind.kAllToAll), 0, 1, 0)]


@pytest.mark.parametrize("name", ["mesh24_8x8", "mesh23_12x18", "mesh222_rank2_small",
                                  "mesh222_rank3_small", "mesh42_1024sq"])
@pytest.mark.parametrize("fuse", [False, True])
def test_all_reference_pairs_small(cuda, name, fuse):
    c = CASES[name]
    pairs = c["pairs"]
    if len(pairs) > 400:
        pairs = random.Random(11).sample(pairs, 400)
    g = O.fill_global(tuple(c["shape"]), c["dtype_bytes"])
    for src, tgt, *_ in pairs:
        check_conversion(c["mesh"], c["shape"], c["dtype_bytes"], src, tgt, fuse, g)


PAIRS_2x4 = ["S01R", "S0S1", "S1S0", "RS01", "RR"]


@pytest.mark.parametrize("fuse", [False, True])
def test_config3_all_20_pairs_on_2x4_8192sq_bf16(cuda, fuse):
    g = O.fill_global((8192, 8192), 2)
    for a in PAIRS_2x4:
        for b in PAIRS_2x4:
            if a != b:
                check_conversion([2, 4], (8192, 8192), 2, a, b, fuse, g)


@pytest.mark.parametrize("fuse", [False, True])
def test_config4_chains_on_2x2x2(cuda, fuse):
    g = O.fill_global((8192, 8192), 2)
    p = check_conversion([2, 2, 2], (8192, 8192), 2, "S012R", "RS012", fuse, g)
    assert len(p.steps) == 5
    check_conversion([2, 2, 2], (8192, 8192), 2, "RS012", "S012R", fuse, g)
    g3 = O.fill_global((512, 512, 256), 2)
    p = check_conversion([2, 2, 2], (512, 512, 256), 2, "S0S1R", "RS1S0", fuse, g3)
    assert len(p.steps) == 1
    check_conversion([2, 2, 2], (512, 512, 256), 2, "RS1S0", "S0S1R", fuse, g3)


@pytest.mark.parametrize("eb", [1, 2, 4, 8])
def test_config2_mesh8_gather_and_all_to_all(cuda, eb):
    shape = (64, 8192 // eb)
    g = O.fill_global(shape, eb)
    for tgt in ["RR", "RS0"]:
        check_conversion([8], shape, eb, "S0R", tgt, False, g)
        check_conversion([8], shape, eb, "S0R", tgt, True, g)


def test_edge_shapes_and_unaligned_runs(cuda):
    cases = [
        ([2, 3], (12, 9), 1, "S0S1", "S10R"),    # 3-byte runs, 1-byte vectors
        ([2, 3], (6, 9), 2, "RS1", "S10R"),
        ([4], (4,), 8, "S0", "R"),               # rank-1, one element per shard
        ([2, 2, 2, 2], (2, 2, 2, 2), 4, "S0S1S2S3", "S3S2S1S0"),  # rank-4, 16 devices
        ([2, 2], (4, 4, 6, 8), 2, "RS0RS1", "S10RRR"),
        ([3], (3, 5), 4, "S0R", "RR"),
        ([1, 4], (4, 4), 4, "S1R", "RS01"),      # unit mesh axis
        ([2, 2], (1, 16), 4, "RS01", "RS10"),    # leading unit dim
    ]
    for mesh, shape, eb, a, b in cases:
        for fuse in (False, True):
            check_conversion(mesh, shape, eb, a, b, fuse)


def test_random_meshes_shapes_and_specs(cuda):
    """300 random conversions: mesh rank 1-3 (non-power-of-two extents
    included), tensor rank 1-4, dtype 1/2/4/8 bytes, random valid specs,
    stepwise and collapsed, bytewise vs the oracle."""
    from test_layout_api import all_valid_specs

    rng = random.Random(20230205)
    meshes = [[2], [3], [4], [8], [2, 2], [2, 3], [3, 2], [2, 4], [4, 2], [2, 2, 2], [1, 4]]
    done = 0
    while done < 300:
        mesh_shape = rng.choice(meshes)
        rank = rng.choice([1, 2, 3, 4])
        shape = tuple(rng.choice([2, 4, 6, 8, 12, 16, 24]) for _ in range(rank))
        eb = rng.choice([1, 2, 4, 8])
        specs = all_valid_specs(TensorMeta(shape, eb), DeviceMesh.uniform(mesh_shape))
        if len(specs) < 2:
            continue
        a, b = rng.choice(specs), rng.choice(specs)
        check_conversion(mesh_shape, shape, eb, str(a), str(b), rng.random() < 0.5)
        done += 1


def test_run_step_for_each_kind(cuda):
    mesh = Mesh.local([2, 4])
    meta = TensorMeta((64, 96), 4)
    g = O.fill_global((64, 96), 4)
    src = ShardingSpec.parse("S0R", 2)
    for tgt in ["RR", "S01R", "RS0"]:  # all-gather, shard-slice, all-to-all
        path = find_transform_path(src, ShardingSpec.parse(tgt, 2), mesh.geo, meta)
        assert len(path.steps) == 1
        ins = to_dev(O.shards(g, [[0], []], [2, 4]))
        t = path.steps[0].result
        outs = [torch.empty(t.local_shape(meta, mesh.geo), dtype=torch.int32, device="cuda")
                for _ in range(8)]
        mesh.run_step(src, path.steps[0], meta, ins, outs)
        want = O.shards(g, O.parse_spec(tgt, 2), [2, 4])
        for o, w in zip(outs, want):
            assert o.cpu().numpy().tobytes() == w.tobytes()


def test_inconsistent_steps_are_rejected(cuda):
    from paper_2302_02599_b200.layout import ArgumentError

    mesh = Mesh.local([2, 4])
    meta = TensorMeta((8, 8), 4)
    path = find_transform_path(ShardingSpec.parse("S01R", 2), ShardingSpec.parse("RR", 2),
                               mesh.geo, meta)
    path.steps = path.steps[::-1]  # gather axis 0 before axis 1: not a valid replay
    ins = [torch.zeros(1, 8, dtype=torch.int32, device="cuda") for _ in range(8)]
    outs = [torch.zeros(8, 8, dtype=torch.int32, device="cuda") for _ in range(8)]
    with pytest.raises(ArgumentError):
        mesh.run_path(path, meta, ins, outs)


def test_nonzero_stream_and_kernel_launch_counter(cuda):
    before = launch_count()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        check_conversion([2, 2], (256, 256), 4, "S0S1", "S1S0", True, stream=s)
    assert launch_count() > before


@pytest.mark.parametrize("dtype,code", [(torch.float32, 0), (torch.bfloat16, 1)])
def test_partial_sum_all_reduce(cuda, dtype, code):
    mesh = Mesh.local([2, 4])
    torch.manual_seed(0)
    parts = [torch.randn(4096 + 8, dtype=dtype, device="cuda") for _ in range(8)]
    host = [p.cpu().view(torch.int16 if code else torch.int32).numpy().copy() for p in parts]
    for axes in ([1], [0], [0, 1]):
        bufs = [p.clone() for p in parts]
        mesh.all_reduce(axes, bufs)
        torch.cuda.synchronize()
        geo = DeviceMesh.uniform([2, 4])
        for d in range(8):
            c = geo.coord_of(d)
            members = [m for m in range(8)
                       if all(geo.coord_of(m)[a] == c[a] for a in range(2) if a not in axes)]
            want = O.group_sum([host[m].view(np.float32 if code == 0 else np.uint16)
                                for m in members], code)
            got = bufs[d].cpu().view(torch.int16 if code else torch.int32).numpy()
            assert got.tobytes() == want.tobytes(), (axes, d)


# Descriptor tables longer than one launch's parameter/shared-memory table
# (40 tile / 64 TMA-ring / 128 LDG descriptors) run as consecutive launches
# over slices of the table: 16-device all-to-alls have 256 pieces. The
# column count picks the engine through the run length (2 KiB rows: TMA bulk
# ring; 256 B: TMA tensor tiles; 32 B: LDG).
# The engines also switch by size (8 MiB: bulk ring; below, the LDG kernel's
# small-launch variant); short strided rows stay on LDG (the tensor-tile
# engine is opt-in, test_tile_engine_forced_parity runs it).
@pytest.mark.parametrize("rows,cols,engine", [(256, 16384, "bulk"), (16384, 2048, "ldg"),
                                              (256, 2048, "ldg"), (256, 256, "ldg")])
def test_many_descriptor_tables_span_launches(cuda, rows, cols, engine):
    import os

    mesh = Mesh.local([16])
    meta = TensorMeta((rows, cols), 2)
    s, t = ShardingSpec.parse("S0R", 1), ShardingSpec.parse("RS0", 1)
    if "APL_COPY_ENGINE" not in os.environ and "APL_TILE_AUTO" not in os.environ:
        assert mesh.exchange_engine(s, t, meta) == engine
    check_conversion([16], (rows, cols), 2, "S0R", "RS0", True)
    check_conversion([4, 4], (rows, cols), 2, "S01R", "RS10", True)


# BASELINE config 2 at full size (1 GiB and 4 GiB bf16 on [8]) -- too big for
# the CPU oracle, so checked on the device through size-independent facts:
# every RR replica equals the concatenation of the S0R shards, every RS0
# shard equals its column block of that concatenation, and S0R->RS0->S0R is
# the identity (bit-exact round trip).
@pytest.mark.parametrize("gib", [1, 4])
def test_config2_full_size_properties(cuda, gib):
    rows = (gib << 30) // (2 * 8192)
    mesh = Mesh.local([8])
    meta = TensorMeta((rows, 8192), 2)
    s0r, rr, rs0 = (ShardingSpec.parse(x, 1) for x in ("S0R", "RR", "RS0"))
    gen = torch.Generator(device="cuda").manual_seed(2302)
    ins = [torch.empty(rows // 8, 8192, dtype=torch.int16, device="cuda") for _ in range(8)]
    for x in ins:
        x.random_(-32768, 32767, generator=gen)
    full = torch.cat(ins)
    a2a = [torch.empty(rows, 1024, dtype=torch.int16, device="cuda") for _ in range(8)]
    mesh.run_path(find_transform_path(s0r, rs0, mesh.geo, meta), meta, ins, a2a, fuse=True)
    torch.cuda.synchronize()
    for q in range(8):
        assert torch.equal(a2a[q], full[:, q * 1024:(q + 1) * 1024]), q
    back = [torch.empty_like(x) for x in ins]
    mesh.run_path(find_transform_path(rs0, s0r, mesh.geo, meta), meta, a2a, back, fuse=True)
    torch.cuda.synchronize()
    for x, y in zip(ins, back):
        assert torch.equal(x, y)
    del a2a, back
    if gib == 1:  # 8 x 1 GiB replicas
        ag = [torch.empty(rows, 8192, dtype=torch.int16, device="cuda") for _ in range(8)]
        mesh.run_path(find_transform_path(s0r, rr, mesh.geo, meta), meta, ins, ag, fuse=True)
        torch.cuda.synchronize()
        for d in range(8):
            assert torch.equal(ag[d], full), d


@pytest.mark.parametrize("engine", ["tile", "bulk", "ldg"])
def test_engine_forced_parity(cuda, engine):
    """Every copy engine, forced for a whole process (the policy is read once
    per process), passes this module's parity tests: the TMA tensor-tile
    engine is opt-in in the automatic policy, so this is where it runs."""
    import os
    import subprocess
    import sys

    if os.environ.get("APL_COPY_ENGINE"):
        pytest.skip("already running under a forced engine")
    env = dict(os.environ, APL_COPY_ENGINE=engine)
    r = subprocess.run([sys.executable, "-m", "pytest", __file__, "-q", "-x", "-m", "gpu",
                        "-k", "not engine_forced_parity and not full_size"],
                       env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
