"""The reference's transformer-block graph (proj/tests/fixtures/gpt_block.json)
executed from the reference planner's own plans (tests/golden/plans/gpt_block_*)
on a simulated mesh, and the block_ops.cu kernels its non-GEMM nodes run on.

Block numerics: bf16 storage at every node, fp32 math; compared with an fp32
torch forward of the same bf16 operands. Tolerance: max|out - ref| / max|ref|
<= 4e-2 and mean|out - ref| / mean|ref| <= 1e-2 (about fifteen bf16 roundings
in sequence). Kernel unit tests: bf16 outputs within 1e-2 relative of fp32
torch; u8 / byte work (embedding rows, transpose, mask) bit-exact.

Elementwise bindings (executor module docstring): mask2 = !mask,
scaled = scores / sqrt(h), att_in = scaled - 1e4 * mask2, act = GELU."""
import json
from pathlib import Path

import pytest
import torch
import torch.nn.functional as F

from paper_2302_02599_b200 import block_ops as B
from paper_2302_02599_b200.executor import MASK_FILL, PlanExecutor
from paper_2302_02599_b200.runtime import Mesh, launch_count

pytestmark = pytest.mark.gpu

PLANS = Path(__file__).resolve().parent / "golden" / "plans"


def _rel(out, ref):
    return ((out.float() - ref.float()).abs().max() / ref.float().abs().max()).item()


# ---- kernels ---------------------------------------------------------------
@pytest.mark.parametrize("rows,width", [(4096, 1024), (333, 64), (17, 1000), (5, 3), (1000, 512),
                                        (300, 2048), (64, 4096)])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_layernorm_softmax(cuda, rows, width, dtype):
    torch.manual_seed(rows + width)
    x = (torch.randn(rows, width, device="cuda") * 3 + 1).to(dtype)
    g = (1 + 0.1 * torch.randn(width, device="cuda")).to(dtype)
    b = (0.1 * torch.randn(width, device="cuda")).to(dtype)
    y = torch.empty_like(x)
    tol = 1e-2 if dtype == torch.bfloat16 else 1e-5
    B.layernorm(x, g, b, y)
    ref = F.layer_norm(x.float(), (width,), g.float(), b.float(), 1e-5)
    assert _rel(y, ref) <= tol
    B.layernorm(x, None, None, y)
    assert _rel(y, F.layer_norm(x.float(), (width,), eps=1e-5)) <= tol
    B.softmax(x, y)
    ref = torch.softmax(x.float(), -1)
    assert ((y.float() - ref).abs().max()).item() <= tol * ref.max().item()
    torch.testing.assert_close(y.float().sum(-1), torch.ones(rows, device="cuda"),
                               atol=2e-2 if dtype == torch.bfloat16 else 1e-5, rtol=0)


def test_softmax_masked_rows(cuda):
    x = torch.randn(64, 256, device="cuda").bfloat16()
    m = (torch.rand(64, 256, device="cuda") < 0.5).to(torch.uint8)
    m[:, 0] = 0  # every row keeps one position
    z = torch.empty_like(x)
    B.add(x, m, z, MASK_FILL)
    y = torch.empty_like(x)
    B.softmax(z, y)
    ref = torch.softmax(x.float().masked_fill(m.bool(), float("-inf")), -1)
    assert (y.float() - ref).abs().max().item() <= 1e-2
    assert (y[m.bool()] == 0).all()


@pytest.mark.parametrize("rows,width", [(8192, 1024), (100, 72), (9, 5)])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_masked_softmax_fused(cuda, rows, width, dtype):
    """softmax(alpha * x + fill * mask) in one pass == the three-node chain
    computed in fp32."""
    x = (torch.randn(rows, width, device="cuda") * 8).to(dtype)
    m = (torch.rand(rows, width, device="cuda") < 0.4).to(torch.uint8)
    m[:, -1] = 0
    y = torch.empty_like(x)
    B.masked_softmax(x, y, 0.125, m, MASK_FILL)
    ref = torch.softmax(0.125 * x.float() + MASK_FILL * m.float(), -1)
    assert (y.float() - ref).abs().max().item() <= (1e-2 if dtype == torch.bfloat16 else 1e-5)
    B.masked_softmax(x, y, 0.5)
    ref = torch.softmax(0.5 * x.float(), -1)
    assert (y.float() - ref).abs().max().item() <= (1e-2 if dtype == torch.bfloat16 else 1e-5)


@pytest.mark.parametrize("n,width,eb", [(8192, 1024, 2), (100, 7, 2), (33, 24, 4), (5, 3, 1)])
def test_embedding_rows_bit_exact(cuda, n, width, eb):
    dt = {1: torch.uint8, 2: torch.bfloat16, 4: torch.float32}[eb]
    vocab = 5000
    table = torch.randint(0, 255, (vocab, width), device="cuda", dtype=torch.uint8).to(dt)
    ids = torch.randint(0, vocab, (n,), device="cuda", dtype=torch.int64)
    ids[0], ids[-1] = vocab - 1, 0
    out = torch.empty(n, width, dtype=dt, device="cuda")
    B.embedding(ids, table, out)
    assert torch.equal(out, table[ids])
    # a hidden-sharded table is a narrower contiguous one
    shard = table[:, : max(1, width // 2)].contiguous()
    o2 = torch.empty(n, shard.shape[1], dtype=dt, device="cuda")
    B.embedding(ids, shard, o2)
    assert torch.equal(o2, shard[ids])
    ids[1] = vocab  # out of range -> zero row
    B.embedding(ids, table, out)
    assert (out[1] == 0).all()


@pytest.mark.parametrize("vb,hb,eb,width", [(8, 1, 2, 1024), (2, 4, 2, 1024), (4, 2, 4, 24),
                                             (2, 2, 2, 6), (1, 8, 1, 40)])
def test_embedding_from_owner_blocks(cuda, vb, hb, eb, width):
    """All-gather fused into the lookup: rows read from the owners' blocks
    give exactly the rows of the gathered table, for any column slice."""
    dt = {1: torch.uint8, 2: torch.bfloat16, 4: torch.float32}[eb]
    vocab, n = 96 * vb, 777
    table = torch.randint(0, 255, (vocab, width), device="cuda", dtype=torch.uint8).to(dt)
    blocks = [table[i * (vocab // vb):(i + 1) * (vocab // vb),
                    j * (width // hb):(j + 1) * (width // hb)].contiguous()
              for i in range(vb) for j in range(hb)]
    ids = torch.randint(0, vocab, (n,), device="cuda", dtype=torch.int64)
    for c0, cols in ((0, width), (width // 2, width // 2), (width - width // hb, width // hb)):
        out = torch.empty(n, cols, dtype=dt, device="cuda")
        B.embedding_blocks(ids, [b.data_ptr() for b in blocks], vb, hb, vocab, width, c0, out)
        assert torch.equal(out, table[ids, c0:c0 + cols])


@pytest.mark.parametrize("shape", [(8, 1024, 1024), (3, 33, 65), (1, 7, 1), (2, 64, 16)])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32, torch.uint8, torch.int64])
def test_transpose_bit_exact(cuda, shape, dtype):
    x = torch.randint(0, 100, shape, device="cuda").to(dtype)
    y = torch.empty(shape[0], shape[2], shape[1], dtype=dtype, device="cuda")
    B.transpose_last2(x, y)
    assert torch.equal(y, x.transpose(1, 2))


@pytest.mark.parametrize("n", [1 << 20, 1001])
def test_elementwise(cuda, n):
    a = torch.randn(n, device="cuda").bfloat16()
    b = torch.randn(n, device="cuda").bfloat16()
    m = (torch.rand(n, device="cuda") < 0.3).to(torch.uint8)
    y = torch.empty_like(a)
    B.scale(a, y, 0.125)
    assert torch.equal(y, (a.float() * 0.125).bfloat16())
    B.add(a, b, y)
    assert torch.equal(y, (a.float() + b.float()).bfloat16())
    B.add(a, m, y, MASK_FILL)
    assert torch.equal(y, (a.float() + MASK_FILL * m.float()).bfloat16())
    mn = torch.empty_like(m)
    B.mask_not(m, mn)
    assert torch.equal(mn, (m == 0).to(torch.uint8))


# ---- the block ---------------------------------------------------------------
def _operands(graph, seed=2302):
    """bf16 parameters, int64 token ids, a causal u8 keep-mask."""
    torch.manual_seed(seed)
    shapes = {n["id"]: n["outputs"][0]["shape"] for n in graph["nodes"] if n["outputs"]}
    b, s = shapes["tok"]
    vocab, h = shapes["wte"]
    f = shapes["w1"][1]
    dev = "cuda"
    p = {
        "tok": torch.randint(0, vocab, (b, s), device=dev, dtype=torch.int64),
        "mask": torch.tril(torch.ones(s, s, device=dev, dtype=torch.uint8)).expand(b, s, s)
        .contiguous(),
        "wte": torch.randn(vocab, h, device=dev).bfloat16(),
        "g1": (1 + 0.1 * torch.randn(h, device=dev)).bfloat16(),
        "b1": (0.1 * torch.randn(h, device=dev)).bfloat16(),
        "g2": (1 + 0.1 * torch.randn(h, device=dev)).bfloat16(),
        "b2": (0.1 * torch.randn(h, device=dev)).bfloat16(),
        "w1": (torch.randn(h, f, device=dev) / h ** 0.5).bfloat16(),
        "w2": (torch.randn(f, h, device=dev) / f ** 0.5).bfloat16(),
    }
    for w in ("wq", "wk", "wv", "wo"):
        p[w] = (torch.randn(h, h, device=dev) / h ** 0.5).bfloat16()
    return p


def block_reference(p):
    """fp32 torch forward of the gpt_block graph (same node order)."""
    f = {k: v.float() if v.is_floating_point() else v for k, v in p.items()}
    b, s = p["tok"].shape
    h = p["wte"].shape[1]
    emb = f["wte"][p["tok"]]
    ln1 = F.layer_norm(emb, (h,), f["g1"], f["b1"], 1e-5).reshape(b * s, h)
    q = (ln1 @ f["wq"]).reshape(b, s, h)
    k = (ln1 @ f["wk"]).reshape(b, s, h)
    v = (ln1 @ f["wv"]).reshape(b, s, h)
    scores = q @ k.transpose(1, 2)
    att_in = scores / h ** 0.5 + MASK_FILL * (p["mask"] == 0).float()
    ctx = torch.softmax(att_in, -1) @ v
    res1 = (ctx.reshape(b * s, h) @ f["wo"]).reshape(b, s, h) + emb
    ln2 = F.layer_norm(res1, (h,), f["g2"], f["b2"], 1e-5).reshape(b * s, h)
    mlp = F.gelu(ln2 @ f["w1"]) @ f["w2"]
    return mlp.reshape(b, s, h) + res1


_CACHE = {}


def _case(tag):
    if tag not in _CACHE:
        graph = json.loads((PLANS / f"gpt_block_{tag}_graph.json").read_text())
        if tag == "fixture":  # the reference's own fp32 [4,16,64] block, run in bf16
            for n in graph["nodes"]:
                for o in n["outputs"]:
                    if o["dtype_bytes"] == 4:
                        o["dtype_bytes"] = 2
        p = _operands(graph)
        _CACHE.clear()
        _CACHE[tag] = (graph, p, block_reference(p))
    return _CACHE[tag]


BLOCK_PLANS = sorted(p.name for p in PLANS.glob("gpt_block_b*_mesh*.json"))
# the reference fixture's own plans: ragged tiny shards (2-row GEMMs, 8-wide
# softmax rows, split-bm / split-bn / emb-h forms) on the same code path
FIXTURE_PLANS = sorted(p.name for p in PLANS.glob("gpt_block_fixture_mesh*.json"))


@pytest.mark.parametrize("name", BLOCK_PLANS + FIXTURE_PLANS)
@pytest.mark.parametrize("fuse", [True, False])
def test_block_plans_execute(cuda, name, fuse):
    graph, feeds, ref = _case(name.split("_mesh")[0].removeprefix("gpt_block_"))
    plan = json.loads((PLANS / name).read_text())
    mesh = Mesh.local(plan["mesh"]["shape"])
    # fuse=False also runs the table all-gather unfused (gather, then lookup)
    ex = PlanExecutor(mesh, graph, plan, fuse=fuse, fuse_gather=None if fuse else False)
    ex.check_against_plan()
    before = launch_count()
    outs = ex.forward(feeds)
    torch.cuda.synchronize()
    assert launch_count() > before
    for o in outs:
        assert o.shape == ref.shape and o.dtype == torch.bfloat16
        assert _rel(o, ref) <= 4e-2
        assert ((o.float() - ref).abs().mean() / ref.abs().mean()).item() <= 1e-2
    for o in outs[1:]:
        assert torch.equal(o, outs[0])


def test_block_plans_agree_bytewise(cuda):
    """Layouts change where the data lives, not the arithmetic of a local
    op: plans whose GEMM / softmax / layernorm shards cover the same rows
    give the same bytes (split-b on [8] vs [2,4] vs [2,2,2] meshes)."""
    graph, feeds, _ = _case("b8s1024")
    outs = []
    for m in ("8", "2x4"):
        plan = json.loads((PLANS / f"gpt_block_b8s1024_mesh{m}_unlimited.json").read_text())
        ex = PlanExecutor(Mesh.local(plan["mesh"]["shape"]), graph, plan)
        outs.append(ex.forward(feeds)[0].clone())
    assert torch.equal(outs[0], outs[1])


def test_attention_chain_fused(cuda):
    """scaled -> att_in -> att runs as one masked-softmax pass when the plan
    keeps the chain in one layout; the unfused chain (train=True forward)
    gives the same block output within bf16 rounding."""
    graph, feeds, ref = _case("b8s1024")
    plan = json.loads((PLANS / "gpt_block_b8s1024_mesh8_unlimited.json").read_text())
    ex = PlanExecutor(Mesh.local(plan["mesh"]["shape"]), graph, plan)
    assert "att" in ex._attn
    shards = {k: ex.shard(k, v) for k, v in feeds.items()}
    n0 = launch_count()
    fused = ex.forward(shards)[0].clone()
    n1 = launch_count()
    plain = ex.forward(shards, train=True)[0].clone()
    n2 = launch_count()
    torch.cuda.synchronize()
    assert n2 - n1 > n1 - n0  # the unfused chain launches more kernels
    assert _rel(fused, plain) <= 2e-2
    assert _rel(fused, ref) <= 4e-2


# ---- backward ----------------------------------------------------------------
@pytest.mark.parametrize("rows,width", [(2048, 1024), (77, 40), (9, 5), (1000, 512), (64, 4096)])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_layernorm_softmax_backward(cuda, rows, width, dtype):
    torch.manual_seed(rows)
    x = (torch.randn(rows, width, device="cuda") * 2 + 0.5).to(dtype)
    g = (1 + 0.1 * torch.randn(width, device="cuda")).to(dtype)
    b = (0.1 * torch.randn(width, device="cuda")).to(dtype)
    dy = torch.randn(rows, width, device="cuda").to(dtype)
    tol = 2e-2 if dtype == torch.bfloat16 else 1e-4
    xf, gf, bf = (t.float().requires_grad_() for t in (x, g, b))
    F.layer_norm(xf, (width,), gf, bf, 1e-5).backward(dy.float())
    dx = torch.empty_like(x)
    dg = torch.zeros(width, device="cuda")
    db = torch.zeros(width, device="cuda")
    B.layernorm_backward(x, g, dy, dx, dg, db)
    assert _rel(dx, xf.grad) <= tol
    assert _rel(dg, gf.grad) <= tol and _rel(db, bf.grad) <= tol
    dg2, db2 = torch.zeros_like(dg), torch.zeros_like(db)  # no atomics: bit-reproducible
    B.layernorm_backward(x, g, dy, dx, dg2, db2)
    assert torch.equal(dg, dg2) and torch.equal(db, db2)
    yf = xf.detach().clone().requires_grad_()
    y = torch.softmax(yf, -1)
    (y * 0.5).backward(dy.float())  # alpha = 0.5 folds the chain's scale
    B.softmax_backward(y.detach().to(dtype), dy, dx, 0.5)
    assert _rel(dx, yf.grad) <= 3 * tol


def test_embedding_backward_accumulates(cuda):
    vocab, width, n = 300, 96, 5000
    ids = torch.randint(0, vocab, (n,), device="cuda", dtype=torch.int64)
    dy = torch.randn(n, width, device="cuda").bfloat16()
    dt = torch.zeros(vocab, width, device="cuda")
    B.embedding_backward(ids, dy, dt)
    ref = torch.zeros(vocab, width, device="cuda").index_add_(0, ids, dy.float())
    torch.testing.assert_close(dt, ref, atol=1e-3, rtol=1e-4)


def test_embedding_backward_owner_block(cuda):
    """Reduce-scatter fused: one owner block of the table gradient from
    several sources' (ids, dy) == that block of the summed full gradient."""
    vocab, width, n, nsrc = 512, 64, 700, 4
    ids = [torch.randint(0, vocab, (n,), device="cuda", dtype=torch.int64) for _ in range(nsrc)]
    dys = [torch.randn(n, width, device="cuda").bfloat16() for _ in range(nsrc)]
    full = torch.zeros(vocab, width, device="cuda")
    for i, d in zip(ids, dys):
        full.index_add_(0, i, d.float())
    for v0, c0, rows, cols in ((0, 0, vocab, width), (128, 0, 128, width), (256, 32, 256, 32)):
        blk = torch.zeros(rows, cols, device="cuda")
        B.embedding_backward_block(ids, dys, blk, v0, c0)
        torch.testing.assert_close(blk, full[v0:v0 + rows, c0:c0 + cols], atol=1e-3, rtol=1e-4)


@pytest.mark.parametrize("a_t,b_t", [(False, False), (False, True), (True, False)])
def test_bmm_layouts(cuda, a_t, b_t):
    """The batched GEMM of batched-matmul nodes and their backward (dA =
    dC.B^T, dB = A^T.dC) on the tcgen05 grouped kernel, fp32 out, vs fp32."""
    nb, m, k, n = 4, 256, 192, 320
    a = torch.randn(nb, k, m, device="cuda").bfloat16() if a_t else \
        torch.randn(nb, m, k, device="cuda").bfloat16()
    b = torch.randn(nb, n, k, device="cuda").bfloat16() if b_t else \
        torch.randn(nb, k, n, device="cuda").bfloat16()
    out = torch.empty(nb, m, n, device="cuda")
    B.bmm(a, b, out, a_t=a_t, b_t=b_t)
    ref = (a.float().transpose(1, 2) if a_t else a.float()) @ \
        (b.float().transpose(1, 2) if b_t else b.float())
    assert _rel(out, ref) <= 1e-5


PARAMS = ("wte", "g1", "b1", "wq", "wk", "wv", "wo", "g2", "b2", "w1", "w2")


def _unshard(ex, nid, shards):
    """Global tensor from a simulated mesh's shards under nid's plan spec."""
    shape, _ = ex.shapes[nid]
    full = torch.empty(shape, dtype=shards[0].dtype, device=shards[0].device)
    spec = ex.spec[nid]
    for d, t in enumerate(shards):
        coord = ex.geo.coord_of(d)
        sl = []
        for k, dim in enumerate(spec.dims):
            s_, split = 0, 1
            for a in dim.axes:
                s_ = s_ * ex.geo.shape[a] + coord[a]
                split *= ex.geo.shape[a]
            L = shape[k] // split
            sl.append(slice(s_ * L, (s_ + 1) * L))
        full[tuple(sl)] = t
    return full


_GRAD_CACHE = {}


def _reference_grads(tag):
    if tag not in _GRAD_CACHE:
        graph, feeds, _ = _case(tag)
        leaves = {k: feeds[k].float().requires_grad_() for k in PARAMS}
        p = dict(feeds)
        p.update(leaves)
        out = block_reference(p)
        torch.manual_seed(7)
        gy = torch.randn(out.shape, device="cuda").bfloat16()
        out.backward(gy.float())
        _GRAD_CACHE.clear()
        _GRAD_CACHE[tag] = (gy, {k: v.grad for k, v in leaves.items()})
    return _GRAD_CACHE[tag]


@pytest.mark.parametrize("name", BLOCK_PLANS + FIXTURE_PLANS)
def test_block_plans_backward(cuda, name):
    """Training step of the block under each reference plan: every
    parameter's gradient (in its plan layout, gathered here for the check)
    against fp32 torch autograd of the same bf16 operands. Tolerance:
    max|g - ref| / max|ref| <= 2e-2 and mean|g - ref| / mean|ref| <= 1.5e-2 per
    parameter (bf16 activations and activation gradients throughout; measured
    <= 0.009 / 0.008, tools/block_grad_check.py)."""
    tag = name.split("_mesh")[0].removeprefix("gpt_block_")
    graph, feeds, _ = _case(tag)
    gy, ref = _reference_grads(tag)
    plan = json.loads((PLANS / name).read_text())
    ex = PlanExecutor(Mesh.local(plan["mesh"]["shape"]), graph, plan)
    ex.forward(feeds, train=True)
    grads = ex.backward(gy)
    torch.cuda.synchronize()
    assert set(grads) == set(PARAMS)
    for k in PARAMS:
        g = _unshard(ex, k, grads[k]).float()
        r = ref[k]
        mx = ((g - r).abs().max() / r.abs().max()).item()
        mean = ((g - r).abs().mean() / r.abs().mean()).item()
        assert mx <= 2e-2 and mean <= 1.5e-2, (k, mx, mean)


# ---- every batched-matmul strategy, backward included --------------------------
def _bmm_case(mesh_shape, st, param_spec):
    """graph: parameters A[4,32,64], B[4,64,64] -> batched-matmul -> output,
    planned with strategy `st` (the catalog's, intraop.cpp:208-231); the
    parameters are stored in `param_spec` (None: the strategy's own input
    layouts, so no conversion runs)."""
    def node(i, kind, inputs, shape=None):
        outs = [{"shape": shape, "dtype_bytes": 2, "requires_grad": True}] if shape else []
        return {"id": i, "kind": kind, "inputs": [[x, 0] for x in inputs], "outputs": outs}

    graph = {"version": 1, "placeholders": [], "output": "out",
             "nodes": [node("A", "parameter", [], [4, 32, 64]),
                       node("B", "parameter", [], [4, 64, 64]),
                       node("mm", "batched-matmul", ["A", "B"]),
                       node("out", "output", ["mm"])]}
    sa = param_spec or str(st.a)
    sb = param_spec or str(st.b)
    plan = {"version": 1, "mesh": {"shape": list(mesh_shape)}, "nodes": {
        "A": {"spec": sa, "strategy": f"src:{sa}", "partial_sum": False},
        "B": {"spec": sb, "strategy": f"src:{sb}", "partial_sum": False},
        "mm": {"spec": str(st.c), "strategy": st.name, "partial_sum": st.partial_sum,
               "reduce_axes": list(st.reduce_axes)},
        "out": {"spec": "RRR", "strategy": "collect", "partial_sum": False}}}
    return graph, plan


def _bmm_strategies():
    from paper_2302_02599_b200 import DeviceMesh, TensorMeta
    from paper_2302_02599_b200.strategies import matmul_strategies

    a, b = TensorMeta((4, 32, 64), 2), TensorMeta((4, 64, 64), 2)
    return [s for s in matmul_strategies(DeviceMesh.uniform([2, 2]), a, b, batched=True)]


@pytest.mark.parametrize("param_spec", [None, "RRR"])
@pytest.mark.parametrize("name", [s.name for s in _bmm_strategies()])
def test_batched_matmul_strategy_backward(cuda, name, param_spec):
    """Forward and backward of one batched matmul under every catalog
    strategy on a 2x2 mesh -- split-k / split-bk / split-mk / split-nk
    (partial sums all-reduced over reduce_axes) included -- against fp32
    torch autograd; with the parameters stored replicated, the input
    conversions and their reverse paths for the gradients run too."""
    st = next(s for s in _bmm_strategies() if s.name == name)
    graph, plan = _bmm_case([2, 2], st, param_spec)
    torch.manual_seed(11)
    A = torch.randn(4, 32, 64, device="cuda").bfloat16()
    Bm = (torch.randn(4, 64, 64, device="cuda") / 8).bfloat16()
    ex = PlanExecutor(Mesh.local([2, 2]), graph, plan)
    out = ex.forward({"A": A, "B": Bm}, train=True)[0]
    af, bf = A.float().requires_grad_(), Bm.float().requires_grad_()
    ref = af @ bf
    assert _rel(out, ref) <= 2e-2
    gy = torch.randn(4, 32, 64, device="cuda").bfloat16()
    ref.backward(gy.float())
    grads = ex.backward(gy)
    torch.cuda.synchronize()
    for k, r in (("A", af.grad), ("B", bf.grad)):
        g = _unshard(ex, k, grads[k]).float()
        assert _rel(g, r) <= 2e-2, (name, k, _rel(g, r))
