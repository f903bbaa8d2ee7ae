"""Backward pass: sharded-matmul gradients, fused GELU
backward, the data-parallel gradient all-reduce and reverse-path gradient
conversions, against torch autograd in fp32 on the same bf16 operands.

Tolerances: max|grad - ref| / max|ref| <= 2e-2 for bf16
gradients and for fp32 weight gradients computed from bf16 intermediates;
<= 1e-5 for the raw tcgen05 GEMMs with fp32 output (MN-major A operand)."""
import json
from pathlib import Path

import pytest
import torch

from paper_2302_02599_b200 import DeviceMesh, ShardingSpec, TensorMeta
from paper_2302_02599_b200.executor import PlanExecutor, megatron_mlp_plan
from paper_2302_02599_b200.runtime import MatmulStrategy, Mesh, gelu, gelu_backward

pytestmark = pytest.mark.gpu

PLANS = Path(__file__).resolve().parent / "golden" / "plans"
GRAPH = json.loads((PLANS / "gpt2_mlp_graph.json").read_text())
TOL = 2e-2


def rel_err(out, ref):
    return ((out.double() - ref.double()).abs().max() / ref.double().abs().max()).item()


def shard(t, spec: ShardingSpec, geo: DeviceMesh, dev: int):
    coord = geo.coord_of(dev)
    sl = []
    for d, dim in enumerate(spec.dims):
        s, split = 0, 1
        for a in dim.axes:
            s = s * geo.shape[a] + coord[a]
            split *= geo.shape[a]
        L = t.shape[d] // split
        sl.append(slice(s * L, (s + 1) * L))
    return t[tuple(sl)].contiguous()


def test_gelu_kernels_match_torch(cuda):
    torch.manual_seed(0)
    x = (torch.randn(1 << 16, device="cuda") * 3).bfloat16()
    dy = torch.randn(1 << 16, device="cuda").bfloat16()
    y = torch.empty_like(x)
    dx = torch.empty_like(x)
    gelu(x, y)
    gelu_backward(dy, x, dx)
    xr = x.float().requires_grad_()
    yr = torch.nn.functional.gelu(xr)
    yr.backward(dy.float())
    torch.cuda.synchronize()
    assert rel_err(y, yr.detach()) <= 1e-2
    assert rel_err(dx, xr.grad) <= 1e-2


# Weight-gradient GEMMs read A as the MN-major operand: check the raw kernel.
@pytest.mark.parametrize("m,n,k", [(256, 384, 512), (1024, 4096, 2048), (136, 200, 80)])
def test_matmul_backward_single_device(cuda, m, n, k):
    mesh = Mesh.local([1])
    p = lambda s: ShardingSpec.parse(s, 1)  # noqa: E731
    st = MatmulStrategy("replicated", p("RR"), p("RR"), p("RR"))
    torch.manual_seed(m)
    a = torch.randn(m, k, device="cuda").bfloat16()
    b = (torch.randn(k, n, device="cuda") / k ** 0.5).bfloat16()
    dc = torch.randn(m, n, device="cuda").bfloat16()
    for b_layout in ("kn", "nk"):
        bs = b if b_layout == "kn" else b.t().contiguous()
        da = torch.empty(m, k, dtype=torch.bfloat16, device="cuda")
        db = torch.empty(bs.shape, dtype=torch.float32, device="cuda")
        mesh.sharded_matmul_backward(st, TensorMeta((m, k), 2), TensorMeta((k, n), 2), [a], [bs],
                                     [dc], [da], [db], b_layout=b_layout)
        torch.cuda.synchronize()
        ref_da = dc.double() @ b.double().t()
        ref_db = a.double().t() @ dc.double()
        assert rel_err(da, ref_da) <= TOL
        assert rel_err(db, ref_db if b_layout == "kn" else ref_db.t()) <= 1e-5


def test_dgelu_epilogue(cuda):
    """dA = (dC . B^T) * GELU'(aux) in the GEMM epilogue."""
    mesh = Mesh.local([1])
    p = lambda s: ShardingSpec.parse(s, 1)  # noqa: E731
    st = MatmulStrategy("replicated", p("RR"), p("RR"), p("RR"))
    m, k, n = 512, 768, 256
    torch.manual_seed(4)
    pre = torch.randn(m, k, device="cuda").bfloat16()
    b = (torch.randn(k, n, device="cuda") / k ** 0.5).bfloat16()
    dc = torch.randn(m, n, device="cuda").bfloat16()
    a = torch.nn.functional.gelu(pre.float()).bfloat16()
    da = torch.empty(m, k, dtype=torch.bfloat16, device="cuda")
    mesh.sharded_matmul_backward(st, TensorMeta((m, k), 2), TensorMeta((k, n), 2), [a], [b], [dc],
                                 [da], None, b_layout="kn", gelu_aux=[pre])
    torch.cuda.synchronize()
    xr = pre.float().requires_grad_()
    torch.nn.functional.gelu(xr).backward(dc.float() @ b.float().t())
    assert rel_err(da, xr.grad) <= TOL


def check_strategy_backward(mesh_shape, st_args, b_layout, m=512, k=256, n=384):
    mesh = Mesh.local(mesh_shape)
    geo, mr = mesh.geo, len(mesh_shape)
    name, a_spec, b_spec, c_spec, red = st_args
    st = MatmulStrategy(name, ShardingSpec.parse(a_spec, mr), ShardingSpec.parse(b_spec, mr),
                        ShardingSpec.parse(c_spec, mr), red)
    torch.manual_seed(7)
    a = torch.randn(m, k, device="cuda").bfloat16()
    b = (torch.randn(k, n, device="cuda") / k ** 0.5).bfloat16()
    dc = torch.randn(m, n, device="cuda").bfloat16()
    nd = mesh.num_devices
    a_sh = [shard(a, st.a, geo, d) for d in range(nd)]
    b_sh = [shard(b, st.b, geo, d) for d in range(nd)]
    if b_layout == "nk":
        b_sh = [t.t().contiguous() for t in b_sh]
    dc_sh = [shard(dc, st.c, geo, d) for d in range(nd)]  # gradient of the reduced C
    da = [torch.empty_like(t) for t in a_sh]
    db = [torch.empty(t.shape, dtype=torch.float32, device="cuda") for t in b_sh]
    mesh.sharded_matmul_backward(st, TensorMeta((m, k), 2), TensorMeta((k, n), 2), a_sh, b_sh,
                                 dc_sh, da, db, b_layout=b_layout)
    torch.cuda.synchronize()
    ref_da = dc.double() @ b.double().t()
    ref_db = a.double().t() @ dc.double()
    for d in range(nd):
        assert rel_err(da[d], shard(ref_da, st.a, geo, d)) <= TOL, (name, d, "dA")
        want = shard(ref_db, st.b, geo, d)
        got = db[d] if b_layout == "kn" else db[d].t()
        assert rel_err(got, want) <= 1e-4, (name, d, "dB")


@pytest.mark.parametrize("case", [
    ([2], ("split-m@0:0", "S0R", "RR", "S0R", [])),
    ([2], ("split-n:0", "RR", "RS0", "RS0", [])),
    ([2], ("split-k:0", "RS0", "S0R", "RR", [0])),
    ([2, 2], ("split-mn@0:0,1", "S0R", "RS1", "S0S1", [])),
    ([2, 2], ("split-mk@0:0,1", "S0S1", "S1R", "S0R", [1])),
    ([2, 2], ("split-nk:0,1", "RS1", "S1S0", "RS0", [1])),
    ([2, 2], ("split-k:01", "RS01", "S01R", "RR", [0, 1])),
    ([2, 4], ("split-mk@0:1,0", "S1S0", "S0R", "S1R", [0])),
    ([8], ("split-m@0:0", "S0R", "RR", "S0R", [])),
])
@pytest.mark.parametrize("b_layout", ["kn", "nk"])
def test_strategy_backward(cuda, case, b_layout):
    mesh_shape, st_args = case
    check_strategy_backward(mesh_shape, st_args, b_layout)


def test_every_catalog_strategy_backward_on_2x2(cuda):
    from paper_2302_02599_b200.strategies import matmul_strategies

    geo = DeviceMesh.uniform([2, 2])
    cat = matmul_strategies(geo, TensorMeta((256, 128), 2), TensorMeta((128, 192), 2))
    for st in cat:
        check_strategy_backward([2, 2], (st.name, str(st.a), str(st.b), str(st.c),
                                         list(st.reduce_axes)), "kn", m=256, k=128, n=192)


@pytest.fixture(scope="module")
def mlp_reference():
    """fp32 autograd of the GPT-2-medium MLP on bf16 operands (config 5)."""
    torch.manual_seed(2302)
    x = torch.randn(16384, 1024, device="cuda").bfloat16()
    w1 = (torch.randn(1024, 4096, device="cuda") / 32).bfloat16()
    w2 = (torch.randn(4096, 1024, device="cuda") / 64).bfloat16()
    gy = torch.randn(16384, 1024, device="cuda").bfloat16()
    xr, w1r, w2r = (t.float().requires_grad_() for t in (x, w1, w2))
    y = torch.nn.functional.gelu(xr @ w1r) @ w2r
    y.backward(gy.float())
    return {"x": x, "w1": w1, "w2": w2}, gy, {"x": xr.grad, "w1": w1r.grad, "w2": w2r.grad}


def run_backward(plan, mlp_reference, fuse=True):
    feeds, gy, ref = mlp_reference
    mesh = Mesh.local(plan["mesh"]["shape"] if "mesh" in plan else [8])
    ex = PlanExecutor(mesh, GRAPH, plan, fuse=fuse)
    ex.forward(feeds, train=True)
    grads = ex.backward(gy, input_grads=True)
    torch.cuda.synchronize()
    assert set(grads) == {"x", "w1", "w2"}
    for nid, shards in grads.items():
        spec = ex.spec[nid]
        for d, g in enumerate(shards):
            want = shard(ref[nid], spec, mesh.geo, d)
            assert g.shape == want.shape, (nid, d)
            assert rel_err(g, want) <= TOL, (nid, d, rel_err(g, want))
    return ex, grads


@pytest.mark.parametrize("name", sorted(p.name for p in PLANS.glob("gpt2_mlp_mesh*.json")))
def test_reference_plans_backward(cuda, mlp_reference, name):
    run_backward(json.loads((PLANS / name).read_text()), mlp_reference)


@pytest.mark.parametrize("fuse", [False, True])
def test_megatron_plan_backward(cuda, mlp_reference, fuse):
    ex, grads = run_backward(megatron_mlp_plan(), mlp_reference, fuse=fuse)
    # x is replicated (RR): its gradient (dX of a split-n fc1, all-reduced over
    # axis 0 in the dA GEMM) is bit-identical on every device.
    for g in grads["x"][1:]:
        assert torch.equal(g, grads["x"][0])


def test_batched_matmul_catalog_backward_on_2x2(cuda):
    """Backward of every batched-matmul strategy (split-b/m/n/k and pairs,
    intraop.cpp:208-231): dA = dC . B^T and dB = A^T . dC per batch element,
    partial sums over the n / m axes reduced (batch axes never are)."""
    from paper_2302_02599_b200.strategies import matmul_strategies

    mesh = Mesh.local([2, 2])
    geo = mesh.geo
    bsz, m, k, n = 8, 256, 128, 192
    torch.manual_seed(11)
    a = torch.randn(bsz, m, k, device="cuda").bfloat16()
    b = (torch.randn(bsz, k, n, device="cuda") / k ** 0.5).bfloat16()
    dc = torch.randn(bsz, m, n, device="cuda").bfloat16()
    ref_da = torch.bmm(dc.double(), b.double().transpose(1, 2))
    ref_db = torch.bmm(a.double().transpose(1, 2), dc.double())
    am, bm = TensorMeta((bsz, m, k), 2), TensorMeta((bsz, k, n), 2)
    cat = matmul_strategies(geo, am, bm, batched=True)
    assert len(cat) > 4
    for st in cat:
        a_sh = [shard(a, st.a, geo, d) for d in range(4)]
        b_sh = [shard(b, st.b, geo, d) for d in range(4)]
        dc_sh = [shard(dc, st.c, geo, d) for d in range(4)]
        da = [torch.empty_like(t) for t in a_sh]
        db = [torch.empty(t.shape, dtype=torch.float32, device="cuda") for t in b_sh]
        mesh.sharded_matmul_backward(st, am, bm, a_sh, b_sh, dc_sh, da, db, b_layout="kn")
        torch.cuda.synchronize()
        for d in range(4):
            assert rel_err(da[d], shard(ref_da, st.a, geo, d)) <= TOL, (st.name, d, "dA")
            assert rel_err(db[d], shard(ref_db, st.b, geo, d)) <= 1e-4, (st.name, d, "dB")
