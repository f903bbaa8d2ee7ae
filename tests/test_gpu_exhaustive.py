"""Exhaustive GPU parity over the reference's own pair enumerations.

Every ordered spec pair the reference enumerates for a mesh (the golden
`paths.json.gz` cases, written by oracle/_ref: mesh222_rank2 = 2,401 pairs,
mesh222_rank3 = 11,236 pairs, mesh24 = 121 pairs) is executed on a simulated
mesh, stepwise along the planner's path and collapsed into one exchange, and
every device's bytes must equal the CPU oracle's direct slicing of the same
global tensor. This is the data-level form of the reference's property tests
(test_layout.cpp:148-165, 264-280; acceptance_test.cpp:124-163), which check
that every enumerated pair has a valid path.

The harness keeps one flat device buffer per spec (all devices' shards back
to back), so a conversion is: fill the output with a sentinel, run, one
torch.equal against the oracle's flat buffer.
"""
import gzip
import json
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import data as O
from paper_2302_02599_b200 import ShardingSpec, TensorMeta, find_transform_path
from paper_2302_02599_b200.runtime import Mesh

pytestmark = pytest.mark.gpu

GOLDEN = Path(__file__).resolve().parent / "golden"
_NP = {1: np.uint8, 2: np.int16, 4: np.int32, 8: np.int64}


def _case(name):
    with gzip.open(GOLDEN / "paths.json.gz", "rt") as f:
        for c in json.load(f)["cases"]:
            if c["name"] == name:
                return c
    raise KeyError(name)


class FlatShards:
    """Oracle shards of one global tensor for every spec, as flat device
    buffers (device d's shard at offset d * per_device_bytes)."""

    def __init__(self, mesh, shape, eb):
        self.mesh, self.shape, self.eb = mesh, tuple(shape), eb
        self.meta = TensorMeta(self.shape, eb)
        self.g = O.fill_global(self.shape, eb)
        self.mr = mesh.geo.rank()
        self.n = mesh.num_devices
        self._want = {}

    def views(self, flat, spec):
        ls = spec.local_shape(self.meta, self.mesh.geo)
        per = int(np.prod(ls)) if ls else 1
        return [flat[d * per:(d + 1) * per].view(ls) for d in range(self.n)]

    def want(self, text):
        if text not in self._want:
            shards = O.shards(self.g, O.parse_spec(text, self.mr), list(self.mesh.geo.shape))
            flat = np.concatenate([np.ascontiguousarray(a).reshape(-1) for a in shards])
            self._want[text] = torch.from_numpy(flat.view(_NP[self.eb])).cuda()
        return self._want[text]


def run_pairs(mesh_shape, shape, eb, pairs, modes=("stepwise", "collapsed")):
    mesh = Mesh.local(mesh_shape)
    fs = FlatShards(mesh, shape, eb)
    outs = {}
    failures, count = [], 0
    stream = torch.cuda.current_stream()
    for src, tgt in pairs:
        s, t = ShardingSpec.parse(src, fs.mr), ShardingSpec.parse(tgt, fs.mr)
        path = find_transform_path(s, t, mesh.geo, fs.meta)
        want = fs.want(tgt)
        if tgt not in outs:
            outs[tgt] = torch.empty_like(want)
        out = outs[tgt]
        ins = fs.views(fs.want(src), s)
        for mode in modes:
            out.fill_(-1)
            mesh.run_path(path, fs.meta, ins, fs.views(out, t), fuse=mode == "collapsed",
                          stream=stream)
            count += 1
            if not torch.equal(out, want):
                failures.append((src, tgt, mode))
    mesh.close()
    return count, failures


@pytest.mark.parametrize("name,shape,eb", [
    ("mesh222_rank2", (16, 16), 2),          # 2,401 pairs (golden written at 8192^2 bf16)
    ("mesh222_rank3", (16, 8, 8), 2),        # 11,236 pairs (golden written at 512x512x256)
    ("mesh24_8192sq_bf16", (8192, 8192), 2),  # 121 pairs at the config-3 size
    ("mesh42_1024sq", (1024, 1024), 4),       # 121 pairs
    ("mesh23_12x18", (12, 18), 4),            # 121 pairs, non-power-of-two axis
])
def test_every_reference_pair(cuda, name, shape, eb):
    c = _case(name)
    pairs = [(p[0], p[1]) for p in c["pairs"]]
    # the data shape must admit every spec the golden enumeration admits
    mesh = Mesh.local(c["mesh"])
    meta = TensorMeta(shape, eb)
    for a in {p[0] for p in pairs}:
        assert ShardingSpec.parse(a, len(c["mesh"])).valid_for(meta, mesh.geo), a
    mesh.close()
    count, failures = run_pairs(c["mesh"], shape, eb, pairs)
    assert count == 2 * len(pairs)
    assert not failures, f"{len(failures)} of {count} conversions differ: {failures[:10]}"
