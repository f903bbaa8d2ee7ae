"""The deep-box rule of the copy-engine policy (runtime.cpp, deep_short_box):
exchanges of >= 64 MiB whose descriptors keep two or more outer dims and
129-256 B runs (or dense 65-128 B source rows into a strided destination)
go to the TMA tensor-tile engine; others stay on the LDG kernel. At the
rule's full size (the 128 MiB [512, 512, 256] bf16 tensor of config 4 on a
simulated 2x2x2 mesh) each conversion's output must equal the CPU oracle's
slicing of the global tensor by the target spec, byte for byte (reference
step semantics layout.cpp:178-219; every-pair timing in
profiles/r02_pairs_222_r3_*.jsonl)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

SHAPE = (512, 512, 256)
CASES = [  # (src, tgt, engine the policy must pick)
    ("RS021R", "S01RS2", "tile"),   # 256 B runs, two outer dims left
    ("S1S20R", "S10RS2", "tile"),
    ("RS12S0", "S012RR", "tile"),
    ("S0S1R", "RS1S0", "ldg"),      # long runs: LDG
    ("S1RR", "RRS0", "ldg"),        # outer dims merge to one: LDG
    ("RRS102", "RS210R", None),     # 64 B runs: no rule
    ("RS1S02", "S120RR", None),
]


@pytest.fixture(scope="module")
def global_tensor():
    from oracle import data as O

    return O.fill_global(SHAPE, 2)


@pytest.mark.parametrize("src,tgt,engine", CASES)
def test_rule_engine_and_bytes(cuda, global_tensor, src, tgt, engine):
    from oracle import data as O
    from paper_2302_02599_b200 import ShardingSpec, TensorMeta, find_transform_path
    from paper_2302_02599_b200.runtime import Mesh

    ms = [2, 2, 2]
    mesh = Mesh.local(ms)
    meta = TensorMeta(SHAPE, 2)
    s, t = ShardingSpec.parse(src, 3), ShardingSpec.parse(tgt, 3)
    got_engine = mesh.exchange_engine(s, t, meta)
    if engine is not None:
        assert got_engine == engine, (src, tgt, got_engine)
    ins = [torch.from_numpy(O.local(global_tensor, O.parse_spec(src, 3), ms, d).view(np.int16))
           .cuda() for d in range(8)]
    want = [O.local(global_tensor, O.parse_spec(tgt, 3), ms, d) for d in range(8)]
    outs = [torch.full(w.shape, -1, dtype=torch.int16, device="cuda") for w in want]
    conv = mesh.prepare(find_transform_path(s, t, mesh.geo, meta), meta, fuse=True)
    conv(ins, outs)
    conv(ins, outs)  # replay: the cached tensor maps
    torch.cuda.synchronize()
    for d in range(8):
        assert outs[d].cpu().numpy().view(want[d].dtype).tobytes() == want[d].tobytes(), (src, tgt, d)
    conv.close()
    mesh.close()
