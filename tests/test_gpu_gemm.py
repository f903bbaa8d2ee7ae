"""tcgen05 GEMM and sharded-matmul strategies vs a plain PyTorch fp32
reference. Tolerance: max|out - ref| / max|ref| <= 2e-2 for
bf16 outputs, <= 1e-5 for fp32 outputs (ref = fp64 product of the same bf16
operands)."""
import pytest
import torch

from paper_2302_02599_b200 import DeviceMesh, ShardingSpec, TensorMeta
from paper_2302_02599_b200.runtime import MatmulStrategy, Mesh, gemm

pytestmark = pytest.mark.gpu

TOL_BF16 = 2e-2
TOL_F32 = 1e-5


def rel_err(out, ref):
    return ((out.double() - ref).abs().max() / ref.abs().max()).item()


def ref_mm(a, bt, gelu=False):
    r = a.double() @ bt.double().t()
    return torch.nn.functional.gelu(r) if gelu else r


@pytest.mark.parametrize("m,n,k", [(128, 128, 64), (256, 512, 1024), (2048, 4096, 1024),
                                   (2048, 1024, 4096), (16384, 512, 1024), (200, 136, 72),
                                   (1, 16, 16), (130, 260, 520)])
@pytest.mark.parametrize("gelu", [False, True])
@pytest.mark.parametrize("b_layout", ["nk", "kn"])
def test_gemm_bf16_out(cuda, m, n, k, gelu, b_layout):
    torch.manual_seed(m + n + k)
    a = torch.randn(m, k, device="cuda").bfloat16()
    bt = (torch.randn(n, k, device="cuda") / k ** 0.5).bfloat16()
    if b_layout == "kn" and (n * 2) % 16:
        pytest.skip("TMA needs 16-byte rows of B[K,N]")
    b = bt.t().contiguous() if b_layout == "kn" else bt
    out = gemm(a, b, gelu=gelu, b_layout=b_layout)
    torch.cuda.synchronize()
    assert rel_err(out, ref_mm(a, bt, gelu)) <= TOL_BF16


@pytest.mark.parametrize("m,n,k", [(256, 256, 256), (1024, 384, 2048), (77, 48, 40)])
def test_gemm_f32_out(cuda, m, n, k):
    torch.manual_seed(1)
    a = torch.randn(m, k, device="cuda").bfloat16()
    bt = torch.randn(n, k, device="cuda").bfloat16()
    out = gemm(a, bt, out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert rel_err(out, ref_mm(a, bt)) <= TOL_F32


def test_gemm_strided_operands(cuda):
    a_full = torch.randn(256, 512, device="cuda").bfloat16()
    b_full = torch.randn(384, 512, device="cuda").bfloat16()
    a, bt = a_full[:, 128:384], b_full[:, 64:320]
    out = torch.zeros(256, 400, device="cuda", dtype=torch.bfloat16)
    gemm(a, bt, out=out[:, :384])
    torch.cuda.synchronize()
    assert rel_err(out[:, :384], ref_mm(a, bt)) <= TOL_BF16
    assert (out[:, 384:] == 0).all()


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


def run_strategy(mesh_shape, name, a_spec, b_spec, c_spec, reduce_axes, m=512, k=256, n=384,
                 gelu=False, out_dtype=torch.bfloat16, b_layout="nk"):
    mesh = Mesh.local(mesh_shape)
    geo, mr = mesh.geo, len(mesh_shape)
    torch.manual_seed(3)
    a = torch.randn(m, k, device="cuda").bfloat16()
    b = (torch.randn(k, n, device="cuda") / k ** 0.5).bfloat16()
    st = MatmulStrategy(name, ShardingSpec.parse(a_spec, mr), ShardingSpec.parse(b_spec, mr),
                        ShardingSpec.parse(c_spec, mr), reduce_axes)
    a_sh = [shard(a, st.a, geo, d) for d in range(mesh.num_devices)]
    if b_layout == "kn":
        bt_sh = [shard(b, st.b, geo, d) for d in range(mesh.num_devices)]
    else:
        bt_sh = [shard(b, st.b, geo, d).t().contiguous() for d in range(mesh.num_devices)]
    c_meta = TensorMeta((m, n), 4 if out_dtype == torch.float32 else 2)
    c_sh = [torch.empty(st.c.local_shape(c_meta, geo), dtype=out_dtype, device="cuda")
            for _ in range(mesh.num_devices)]
    mesh.sharded_matmul(st, TensorMeta((m, k), 2), TensorMeta((k, n), 2), a_sh, bt_sh, c_sh,
                        gelu=gelu, b_layout=b_layout)
    torch.cuda.synchronize()
    ref = a.double() @ b.double()
    if gelu:
        ref = torch.nn.functional.gelu(ref)
    tol = TOL_F32 * 10 if out_dtype == torch.float32 else TOL_BF16
    for d in range(mesh.num_devices):
        want = shard(ref, st.c, geo, d)
        assert rel_err(c_sh[d], want) <= tol, (name, d)


# Reference catalog forms on mesh [2] / [2,2] (proj/src/intraop.cpp:141-234).
@pytest.mark.parametrize("case", [
    ([2], "split-m@0:0", "S0R", "RR", "S0R", []),
    ([2], "split-n:0", "RR", "RS0", "RS0", []),
    ([2], "split-k:0", "RS0", "S0R", "RR", [0]),
    ([2, 2], "split-mn@0:0,1", "S0R", "RS1", "S0S1", []),
    ([2, 2], "split-mk@0:0,1", "S0S1", "S1R", "S0R", [1]),
    ([2, 2], "split-nk:0,1", "RS1", "S1S0", "RS0", [1]),
    ([2, 2], "split-k:01", "RS01", "S01R", "RR", [0, 1]),
    ([2, 2], "split-m@0:01", "S01R", "RR", "S01R", []),
    ([2, 4], "split-mk@0:1,0", "S1S0", "S0R", "S1R", [0]),
])
@pytest.mark.parametrize("gelu", [False, True])
@pytest.mark.parametrize("b_layout", ["nk", "kn"])
def test_sharded_matmul_strategies(cuda, case, gelu, b_layout):
    mesh_shape, name, a, b, c, red = case
    run_strategy(mesh_shape, name, a, b, c, red, gelu=gelu, b_layout=b_layout)


def test_every_catalog_strategy_on_2x2(cuda):
    """All reference-catalog matmul strategies on mesh [2,2] (decoded by
    matmul_strategies, intraop.cpp:141-234) execute to the same product."""
    from paper_2302_02599_b200.strategies import matmul_strategies

    mesh = Mesh.local([2, 2])
    geo = mesh.geo
    m, k, n = 256, 128, 192
    torch.manual_seed(9)
    a = torch.randn(m, k, device="cuda").bfloat16()
    b = (torch.randn(k, n, device="cuda") / k ** 0.5).bfloat16()
    ref = a.double() @ b.double()
    cat = matmul_strategies(geo, TensorMeta((m, k), 2), TensorMeta((k, n), 2))
    assert len(cat) == 16
    for st in cat:
        a_sh = [shard(a, st.a, geo, d) for d in range(4)]
        b_sh = [shard(b, st.b, geo, d) for d in range(4)]
        c_sh = [torch.empty(st.c.local_shape(TensorMeta((m, n), 2), geo), dtype=torch.bfloat16,
                            device="cuda") for _ in range(4)]
        mesh.sharded_matmul(st, TensorMeta((m, k), 2), TensorMeta((k, n), 2), a_sh, b_sh, c_sh,
                            b_layout="kn")
        torch.cuda.synchronize()
        for d in range(4):
            assert rel_err(c_sh[d], shard(ref, st.c, geo, d)) <= TOL_BF16, st.name


def test_batched_matmul_catalog_on_2x2(cuda):
    """Batched-matmul strategies (split-b/m/n/k and pairs, intraop.cpp:208-231)
    run as batched tcgen05 GEMMs on the shards."""
    from paper_2302_02599_b200.strategies import matmul_strategies

    mesh = Mesh.local([2, 2])
    geo = mesh.geo
    bsz, m, k, n = 16, 128, 64, 96
    torch.manual_seed(10)
    a = torch.randn(bsz, m, k, device="cuda").bfloat16()
    b = (torch.randn(bsz, k, n, device="cuda") / k ** 0.5).bfloat16()
    ref = torch.bmm(a.double(), b.double())
    am, bm, cm = TensorMeta((bsz, m, k), 2), TensorMeta((bsz, k, n), 2), TensorMeta((bsz, m, n), 2)
    cat = matmul_strategies(geo, am, bm, batched=True)
    assert any(s.name.startswith("split-bk") for s in cat)
    for st in cat:
        a_sh = [shard(a, st.a, geo, d) for d in range(4)]
        b_sh = [shard(b, st.b, geo, d) for d in range(4)]
        c_sh = [torch.empty(st.c.local_shape(cm, geo), dtype=torch.bfloat16, device="cuda")
                for _ in range(4)]
        mesh.sharded_matmul(st, am, bm, a_sh, b_sh, c_sh, b_layout="kn")
        torch.cuda.synchronize()
        for d in range(4):
            assert rel_err(c_sh[d], shard(ref, st.c, geo, d)) <= TOL_BF16, st.name


def test_split_k_fp32_partials(cuda):
    run_strategy([4], "split-k:0", "RS0", "S0R", "RR", [0], out_dtype=torch.float32)


def test_megatron_mlp_on_mesh8(cuda):
    """Config 5 pinned selection: fc1 split-n:0 (+GELU), fc2 split-k:0 (+AR)."""
    mesh = Mesh.local([8])
    geo = mesh.geo
    torch.manual_seed(5)
    x = torch.randn(2048, 1024, device="cuda").bfloat16()
    w1 = (torch.randn(1024, 4096, device="cuda") / 32).bfloat16()
    w2 = (torch.randn(4096, 1024, device="cuda") / 64).bfloat16()
    p = lambda s: ShardingSpec.parse(s, 1)  # noqa: E731
    fc1 = MatmulStrategy("split-n:0", p("RR"), p("RS0"), p("RS0"))
    fc2 = MatmulStrategy("split-k:0", p("RS0"), p("S0R"), p("RR"), [0])
    xs = [x] * 8
    w1t = [shard(w1, fc1.b, geo, d).t().contiguous() for d in range(8)]
    w2t = [shard(w2, fc2.b, geo, d).t().contiguous() for d in range(8)]
    h = [torch.empty(2048, 512, dtype=torch.bfloat16, device="cuda") for _ in range(8)]
    y = [torch.empty(2048, 1024, dtype=torch.bfloat16, device="cuda") for _ in range(8)]
    mesh.sharded_matmul(fc1, TensorMeta((2048, 1024), 2), TensorMeta((1024, 4096), 2), xs, w1t, h,
                        gelu=True)
    # same fc1 with the weight kept in its logical [k, n] layout (MN-major B)
    w1s = [shard(w1, fc1.b, geo, d) for d in range(8)]
    h_kn = [torch.empty_like(t) for t in h]
    mesh.sharded_matmul(fc1, TensorMeta((2048, 1024), 2), TensorMeta((1024, 4096), 2), xs, w1s,
                        h_kn, gelu=True, b_layout="kn")
    mesh.sharded_matmul(fc2, TensorMeta((2048, 4096), 2), TensorMeta((4096, 1024), 2), h, w2t, y)
    torch.cuda.synchronize()
    ref = torch.nn.functional.gelu(x.float() @ w1.float()) @ w2.float()
    for d in range(8):
        assert rel_err(y[d], ref.double()) <= TOL_BF16
        assert torch.equal(y[d], y[0])  # all-reduce leaves identical replicas
        assert rel_err(h_kn[d], h[d].double()) <= 1e-2


# Every launch plan (1-CTA / CTA-pair kernel x N tile 128 / 256 x whole
# tiles / stream-K / aligned split-K 2 and 4, forced through
# apl_gemm_force_plan) on shapes that under-fill the SMs, ragged tails and
# both B layouts. A split the shape cannot take falls back to a whole-tile plan.
PLANS = [(p, bn, sk) for p in (0, 1) for bn in (128, 256) for sk in (0, 1, 2, 4)]


@pytest.fixture
def force_plan():
    from paper_2302_02599_b200 import _capi as A

    lib = A.lib()
    yield lambda p, bn, sk: lib.apl_gemm_force_plan(p, bn, sk)
    lib.apl_gemm_force_plan(-1, -1, -1)


@pytest.mark.parametrize("plan", PLANS, ids=[f"pair{p}-bn{bn}-sk{sk}" for p, bn, sk in PLANS])
@pytest.mark.parametrize("m,n,k", [(2048, 1024, 4096), (1024, 512, 2048), (384, 768, 1000),
                                   (2048, 1024, 512), (16384, 512, 1024), (300, 200, 136)])
def test_gemm_every_plan(cuda, force_plan, plan, m, n, k):
    assert force_plan(*plan) == 0
    torch.manual_seed(m + k)
    a = torch.randn(m, k, device="cuda").bfloat16()
    bt = (torch.randn(n, k, device="cuda") / k ** 0.5).bfloat16()
    for gelu in (False, True):
        for _ in range(2):  # the second call reuses the stream's workspace and flags
            out = gemm(a, bt, gelu=gelu)
            torch.cuda.synchronize()
            assert rel_err(out, ref_mm(a, bt, gelu)) <= TOL_BF16, (plan, gelu)
    out32 = gemm(a, bt, out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert rel_err(out32, ref_mm(a, bt)) <= TOL_F32, plan
    if (n * 2) % 16 == 0:
        out_kn = gemm(a, bt.t().contiguous(), b_layout="kn", out_dtype=torch.float32)
        torch.cuda.synchronize()
        assert rel_err(out_kn, ref_mm(a, bt)) <= TOL_F32, plan
