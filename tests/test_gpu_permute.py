"""General transpose (any `perm`) and softmax over any `axis` -- the graph
format's full transpose / softmax attributes (reference graph_ir.cpp:270-290;
softmax strategies keep the axis replicated, intraop.cpp:368-384):

* apl_permute against torch.permute, bit for bit, every permutation of
  ranks 2-4 (and a rank-5 sample), 1/2/4/8-byte elements, ragged extents,
  both kernel paths (row copy when the last dim stays, 32x32 tiles else);
* apl_softmax_axis and its backward against fp32 torch;
* the reference planner's own plans for a graph using both
  (tests/golden/make_permute_plans.py: layernorm -> transpose [1,0,2] ->
  softmax axis 1 -> transpose [2,0,1]) on [4] and [2,2], forward and
  backward, against torch autograd."""
import itertools
import json
from pathlib import Path

import pytest
import torch

from paper_2302_02599_b200 import block_ops as B

pytestmark = pytest.mark.gpu
PLANS = Path(__file__).resolve().parent / "golden" / "plans"

SHAPES = {2: [(33, 70), (64, 8), (1, 5)],
          3: [(5, 33, 70), (8, 64, 16), (3, 1, 40)],
          4: [(3, 5, 33, 18), (2, 8, 16, 8)]}
DTYPES = [torch.uint8, torch.int16, torch.float32, torch.int64]


def _rand(shape, dt):
    if dt.is_floating_point:
        return torch.randn(shape, device="cuda", dtype=dt)
    hi = 255 if dt == torch.uint8 else 30000
    return torch.randint(0, hi, shape, device="cuda", dtype=dt)


@pytest.mark.parametrize("rank", [2, 3, 4])
@pytest.mark.parametrize("dt", DTYPES)
def test_permute_every_perm_bit_exact(cuda, rank, dt):
    for shape in SHAPES[rank]:
        x = _rand(shape, dt)
        for perm in itertools.permutations(range(rank)):
            want = x.permute(perm).contiguous()
            y = torch.empty_like(want)
            B.permute(x, y, perm)
            assert torch.equal(y, want), (shape, perm, dt)


def test_permute_rank5_and_offsets(cuda):
    x = _rand((2, 3, 4, 5, 24), torch.int16)
    for perm in [(4, 3, 2, 1, 0), (1, 0, 2, 3, 4), (0, 2, 4, 1, 3), (3, 0, 1, 4, 2)]:
        want = x.permute(perm).contiguous()
        y = torch.empty_like(want)
        B.permute(x, y, perm)
        assert torch.equal(y, want), perm
    # a row-copy permutation on a sliced (non-16-byte-aligned) source: scalar path
    base = _rand((4 * 6 * 10 + 1,), torch.int16)
    x = base[1:].view(4, 6, 10)
    want = x.permute(1, 0, 2).contiguous()
    y = torch.empty_like(want)
    B.permute(x, y, (1, 0, 2))
    assert torch.equal(y, want)


def test_permute_rejects_bad_perm(cuda):
    x = _rand((4, 5), torch.float32)
    with pytest.raises(ValueError):
        B.permute(x, torch.empty(5, 4, device="cuda"), (0, 0))


@pytest.mark.parametrize("dt", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("shape,axis", [((6, 37, 20), 1), ((6, 37, 20), 0), ((6, 37, 20), -2),
                                        ((3, 4, 5, 64), 2), ((3, 4, 5, 64), -1), ((128, 3), 0)])
def test_softmax_axis_forward_backward(cuda, dt, shape, axis):
    torch.manual_seed(0)
    x = (torch.randn(shape, device="cuda") * 3).to(dt)
    y = torch.empty_like(x)
    B.softmax_axis(x, y, axis)
    xr = x.float().requires_grad_(True)
    ref = torch.softmax(xr, axis)
    tol = 8e-3 if dt == torch.bfloat16 else 1e-5
    assert (y.float() - ref).abs().max().item() <= tol
    dy = torch.randn(shape, device="cuda").to(dt)
    ref.backward(dy.float())
    dx = torch.empty_like(x)
    B.softmax_axis_backward(y, dy, dx, axis)
    err = ((dx.float() - xr.grad).abs().max() / xr.grad.abs().max()).item()
    assert err <= (2e-2 if dt == torch.bfloat16 else 1e-4), err


def _reference(feeds, gy=None):
    x = feeds["x"].float()
    g = feeds["g"].float().requires_grad_(True)
    b = feeds["bb"].float().requires_grad_(True)
    ln = torch.nn.functional.layer_norm(x, (x.shape[-1],), g, b, 1e-5)
    out = torch.softmax(ln.permute(1, 0, 2), 1).permute(2, 0, 1)
    if gy is not None:
        out.backward(gy.float())
    return out.detach(), g.grad, b.grad


@pytest.mark.parametrize("mesh_tag", ["4", "2x2"])
def test_permute_softmax_axis_plans(cuda, mesh_tag):
    from paper_2302_02599_b200.executor import PlanExecutor
    from paper_2302_02599_b200.runtime import Mesh

    graph = json.loads((PLANS / "permute_graph.json").read_text())
    plan = json.loads((PLANS / f"permute_mesh{mesh_tag}_unlimited.json").read_text())
    torch.manual_seed(11)
    shapes = {n["id"]: n["outputs"][0]["shape"] for n in graph["nodes"] if n["outputs"]}
    feeds = {"x": torch.randn(shapes["x"], device="cuda").bfloat16(),
             "g": (1 + 0.1 * torch.randn(shapes["g"], device="cuda")).bfloat16(),
             "bb": (0.1 * torch.randn(shapes["bb"], device="cuda")).bfloat16()}
    ex = PlanExecutor(Mesh.local(plan["mesh"]["shape"]), graph, plan)
    ex.check_against_plan()
    outs = ex.forward(feeds, train=True)
    torch.cuda.synchronize()
    torch.manual_seed(12)
    gy = torch.randn(outs[0].shape, device="cuda").bfloat16()
    ref, rg, rb = _reference(feeds, gy)
    for o in outs:
        assert o.shape == ref.shape
        assert (o.float() - ref).abs().max().item() <= 8e-3
    grads = ex.backward(gy)
    torch.cuda.synchronize()
    import sys
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from test_gpu_block import _unshard

    # beta shifts every softmax input of a column alike, so its true gradient
    # is 0 (the reference's is rounding noise): both are measured against
    # gamma's gradient scale
    scale = rg.abs().max()
    for k, r in (("g", rg), ("bb", rb)):
        gk = _unshard(ex, k, grads[k]).float()
        err = ((gk - r).abs().max() / scale).item()
        assert err <= 2e-2, (k, err)
