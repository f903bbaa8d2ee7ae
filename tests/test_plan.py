"""Host-side exchange planning (libapl.so, no GPU): the direct src->tgt
redistribution every fused conversion and the distributed executor use.

Checked on CPU by executing the plan with numpy over simulated devices and
comparing against the oracle, plus the structural properties the runtime
relies on (exact tiling, sender/receiver agreement, minimal bytes,
traffic confined to the source's axis groups)."""
import gzip
import json
import random
from pathlib import Path

import numpy as np
import pytest

from oracle import data as O
from paper_2302_02599_b200 import (DeviceMesh, ShardingSpec, TensorMeta, plan_pieces)

GOLDEN = Path(__file__).resolve().parent / "golden"


def _cases():
    with gzip.open(GOLDEN / "paths.json.gz", "rt") as f:
        return {c["name"]: c for c in json.load(f)["cases"]}


CASES = _cases()


def execute_plan(mesh_shape, shape, src, tgt, ins):
    mesh = DeviceMesh.uniform(mesh_shape)
    mr = len(mesh_shape)
    s, t = ShardingSpec.parse(src, mr), ShardingSpec.parse(tgt, mr)
    meta = TensorMeta(tuple(shape), ins[0].itemsize)
    lt = t.local_shape(meta, mesh)
    outs = []
    for q in range(mesh.num_devices()):
        out = np.full(lt, 0, dtype=ins[0].dtype)
        seen = np.zeros(lt, dtype=np.int32)
        for p in plan_pieces(mesh, s, t, meta, q, "recv"):
            assert p.receiver == q
            ssl = tuple(slice(a, a + e) for a, e in zip(p.src_lo, p.ext))
            dsl = tuple(slice(a, a + e) for a, e in zip(p.dst_lo, p.ext))
            out[dsl] = ins[p.sender][ssl]
            seen[dsl] += 1
        assert (seen == 1).all(), "target block must be tiled exactly once"
        outs.append(out)
    return outs


@pytest.mark.parametrize("name", ["mesh24_8x8", "mesh23_12x18", "mesh222_rank2_small",
                                  "mesh222_rank3_444", "mesh42_1024sq"])
def test_plan_execution_matches_oracle(name):
    c = CASES[name]
    mesh, shape, eb = c["mesh"], tuple(c["shape"]), c["dtype_bytes"]
    g = O.fill_global(shape, eb)
    rng = random.Random(7)
    pairs = c["pairs"] if len(c["pairs"]) <= 200 else rng.sample(c["pairs"], 200)
    for src, tgt, *_ in pairs:
        ins = O.shards(g, O.parse_spec(src, len(mesh)), mesh)
        want = O.shards(g, O.parse_spec(tgt, len(mesh)), mesh)
        got = execute_plan(mesh, shape, src, tgt, ins)
        for a, b in zip(got, want):
            assert a.tobytes() == b.tobytes(), (src, tgt)


def test_sender_and_receiver_views_agree_and_traffic_is_minimal():
    c = CASES["mesh222_rank3_444"]
    mesh = DeviceMesh.uniform(c["mesh"])
    meta = TensorMeta(tuple(c["shape"]), 4)
    rng = random.Random(3)
    for src, tgt, *_ in rng.sample(c["pairs"], 300):
        s, t = ShardingSpec.parse(src, 3), ShardingSpec.parse(tgt, 3)
        recv, send = {}, {}
        for d in range(8):
            for p in plan_pieces(mesh, s, t, meta, d, "recv"):
                recv[(p.sender, p.receiver)] = p
            for p in plan_pieces(mesh, s, t, meta, d, "send"):
                send[(p.sender, p.receiver)] = p
        assert recv.keys() == send.keys()
        for k in recv:
            assert (recv[k].src_lo, recv[k].dst_lo, recv[k].ext) == \
                (send[k].src_lo, send[k].dst_lo, send[k].ext)
        used = set(s.used_axes())
        for (snd, rcv), p in recv.items():
            cs, cr = mesh.coord_of(snd), mesh.coord_of(rcv)
            # senders only differ from receivers on axes the source uses
            assert all(cs[a] == cr[a] for a in range(3) if a not in used)
        # minimal: a device never receives bytes it already holds
        for d in range(8):
            own = [p for (snd, rcv), p in recv.items() if rcv == d and snd == d]
            need_remote = sum(int(np.prod(p.ext)) for (snd, rcv), p in recv.items()
                              if rcv == d and snd != d)
            total = int(np.prod(t.local_shape(meta, mesh)))
            held = sum(int(np.prod(p.ext)) for p in own)
            assert need_remote == total - held


def test_appendix_b_minimal_bytes():
    """SURVEY Appendix B 'min MiB' column (max over GPUs of bytes received)."""
    table = [([2, 4], (8192, 8192), 2, "S01R", "S0S1", 12), ([2, 4], (8192, 8192), 2, "S01R", "S1S0", 16),
             ([2, 4], (8192, 8192), 2, "S01R", "RS01", 14), ([2, 4], (8192, 8192), 2, "S0S1", "S1S0", 16),
             ([2, 4], (8192, 8192), 2, "S01R", "RR", 112), ([2, 4], (8192, 8192), 2, "RR", "S01R", 0),
             ([2, 2, 2], (8192, 8192), 2, "S012R", "RS012", 14),
             ([2, 2, 2], (512, 512, 128), 2, "S0S1R", "RS1S0", 8),
             ([8], (8192, 8192), 4, "S0R", "RR", 224), ([8], (8192, 8192), 4, "S0R", "RS0", 28)]
    for mesh_shape, shape, eb, src, tgt, mib in table:
        mesh = DeviceMesh.uniform(mesh_shape)
        meta = TensorMeta(shape, eb)
        s, t = ShardingSpec.parse(src, len(mesh_shape)), ShardingSpec.parse(tgt, len(mesh_shape))
        worst = 0
        for d in range(mesh.num_devices()):
            b = sum(int(np.prod(p.ext)) * eb for p in plan_pieces(mesh, s, t, meta, d, "recv")
                    if p.sender != d)
            worst = max(worst, b)
        assert worst == mib << 20, (src, tgt, worst / 2**20)
