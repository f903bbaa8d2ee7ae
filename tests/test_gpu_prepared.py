"""Prepared conversions (apl_conversion_*) give the same bytes as
apl_run_path, stepwise and collapsed, and can be captured into a CUDA graph
(no host sync, no allocation after the first run)."""
import pytest
import torch

from oracle import data as O
from paper_2302_02599_b200 import ShardingSpec, TensorMeta, find_transform_path
from paper_2302_02599_b200.runtime import Mesh

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", [([2, 4], (512, 384), "S01R", "S1S0"),
                                  ([2, 2, 2], (256, 256), "S012R", "RS012"),
                                  ([8], (1024, 256), "S0R", "RR")])
@pytest.mark.parametrize("fuse", [False, True])
def test_prepared_matches_oracle_and_graph_replay(cuda, case, fuse):
    mesh_shape, shape, a, b = case
    mesh = Mesh.local(mesh_shape)
    mr = len(mesh_shape)
    meta = TensorMeta(shape, 2)
    g = O.fill_global(shape, 2)
    s, t = ShardingSpec.parse(a, mr), ShardingSpec.parse(b, mr)
    conv = mesh.prepare(find_transform_path(s, t, mesh.geo, meta), meta, fuse=fuse)
    ins = [torch.from_numpy(x).cuda() for x in O.shards(g, O.parse_spec(a, mr), mesh_shape)]
    outs = [torch.full(t.local_shape(meta, mesh.geo), -1, dtype=torch.int16, device="cuda")
            for _ in range(mesh.num_devices)]
    want = O.shards(g, O.parse_spec(b, mr), mesh_shape)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        conv(ins, outs, stream=side)  # first run compiles the device tables
        side.synchronize()
        for o, w in zip(outs, want):
            assert o.cpu().numpy().tobytes() == w.tobytes()
        for o in outs:
            o.fill_(-1)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=side):
            conv(ins, outs, stream=side)
    torch.cuda.current_stream().wait_stream(side)
    graph.replay()
    torch.cuda.synchronize()
    for o, w in zip(outs, want):
        assert o.cpu().numpy().tobytes() == w.tobytes()
