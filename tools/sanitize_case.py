"""Small invocations of every kernel family, for compute-sanitizer (SURVEY §5
race/memory checking). Each case checks its own result, so a run that is
clean under memcheck is also a correct run.

    compute-sanitizer --tool memcheck --error-exitcode 9 \
        python tools/sanitize_case.py {copies|gemm|block|peer}

copies: conversions on simulated 2x4 / 2x2x2 meshes (stepwise and collapsed,
        odd shapes that take the masked tails) vs the C oracle, once per copy
        engine (APL_COPY_ENGINE is set by the caller: ldg | bulk | tile);
        plus the fused all-reduce.
gemm:   tcgen05 GEMMs: 1-CTA (BN 128 / 256), CTA pair, K/M/N tails, GELU
        epilogues, MN-major operands, fused split-k reduce, scatter epilogue.
block:  layernorm / softmax / masked softmax / transpose / embedding forward
        and backward.
peer:   the fused peer exchange (flags + pull + done) with P ranks in this
        process (tools/peer_loopback.py's harness), vs the oracle.
"""
import ctypes as C
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

_NP = {1: np.uint8, 2: np.int16, 4: np.int32, 8: np.int64}


def copies():
    from oracle import data as O
    from paper_2302_02599_b200 import ShardingSpec, TensorMeta, find_transform_path
    from paper_2302_02599_b200.runtime import Mesh

    cases = [([2, 4], (64, 96), 2, "S01R", "RS01"), ([2, 4], (40, 24), 4, "S0S1", "S1S0"),
             ([2, 4], (64, 64), 2, "RR", "S01R"), ([2, 2, 2], (32, 16, 8), 2, "S0S1R", "RS1S0"),
             ([2, 2, 2], (64, 64), 2, "S012R", "RS012"), ([8], (8, 1000), 1, "S0R", "RR"),
             ([8], (64, 24), 8, "S0R", "RS0")]
    for mesh_shape, shape, eb, a, b in cases:
        mesh = Mesh.local(mesh_shape)
        mr = len(mesh_shape)
        meta = TensorMeta(shape, eb)
        s, t = ShardingSpec.parse(a, mr), ShardingSpec.parse(b, mr)
        path = find_transform_path(s, t, mesh.geo, meta)
        g = O.fill_global(shape, eb)
        ins = [torch.from_numpy(np.ascontiguousarray(x).view(_NP[eb])).cuda()
               for x in O.shards(g, O.parse_spec(a, mr), mesh_shape)]
        want = O.shards(g, O.parse_spec(b, mr), mesh_shape)
        for fuse in (False, True):
            outs = [torch.empty(t.local_shape(meta, mesh.geo), dtype=ins[0].dtype, device="cuda")
                    for _ in range(mesh.num_devices)]
            mesh.run_path(path, meta, ins, outs, fuse=fuse)
            torch.cuda.synchronize()
            for o, w in zip(outs, want):
                assert o.cpu().numpy().tobytes() == w.tobytes(), (a, b, fuse)
    mesh = Mesh.local([2, 4])
    parts = [torch.randn(3000, device="cuda") for _ in range(8)]
    ref = torch.stack([p.double() for p in parts]).view(2, 4, -1).sum(0)
    mesh.all_reduce([0], parts)
    torch.cuda.synchronize()
    for d in range(8):
        assert torch.allclose(parts[d].double(), ref[d % 4], atol=1e-5)


def gemm():
    from paper_2302_02599_b200.runtime import gemm as G

    torch.manual_seed(0)
    for m, n, k in [(128, 128, 64), (200, 136, 72), (256, 512, 128), (512, 512, 256),
                    (130, 264, 104)]:
        a = torch.randn(m, k, device="cuda").bfloat16()
        bt = torch.randn(n, k, device="cuda").bfloat16()
        ref = a.float() @ bt.float().t()
        for gelu in (False, True):
            for pair in ("0", "1") if m >= 256 and n >= 256 else ("0",):
                os.environ["APL_GEMM_PAIR"] = pair  # read once; first value sticks
                c = G(a, bt, gelu=gelu, out_dtype=torch.float32)
                want = torch.nn.functional.gelu(ref) if gelu else ref
                err = ((c - want).abs().max() / want.abs().max()).item()
                assert err < 1e-2, (m, n, k, gelu, err)
        c = G(a, bt.t().contiguous(), b_layout="kn", out_dtype=torch.float32)
        assert ((c - ref).abs().max() / ref.abs().max()).item() < 1e-2
    # fused split-k reduce on a simulated mesh (partial sums in one launch)
    from paper_2302_02599_b200 import TensorMeta
    from paper_2302_02599_b200.runtime import Mesh
    from paper_2302_02599_b200.strategies import find_matmul_strategy

    mesh = Mesh.local([4])
    xm, wm = TensorMeta((256, 512), 2), TensorMeta((512, 256), 2)
    strat = find_matmul_strategy("split-k:0", mesh.geo, xm, wm)
    x = torch.randn(256, 512, device="cuda").bfloat16()
    w = torch.randn(512, 256, device="cuda").bfloat16()
    xs = [x[:, 128 * i:128 * (i + 1)].contiguous() for i in range(4)]
    ws = [w[128 * i:128 * (i + 1)].contiguous() for i in range(4)]
    outs = [torch.empty(256, 256, device="cuda", dtype=torch.float32) for _ in range(4)]
    mesh.sharded_matmul(strat, xm, wm, xs, ws, outs, b_layout="kn")
    torch.cuda.synchronize()
    ref = x.float() @ w.float()
    for o in outs:
        assert ((o - ref).abs().max() / ref.abs().max()).item() < 1e-2


def block():
    from paper_2302_02599_b200 import block_ops as B

    torch.manual_seed(1)
    x = torch.randn(70, 200, device="cuda").bfloat16()
    g = torch.randn(200, device="cuda").bfloat16()
    b = torch.randn(200, device="cuda").bfloat16()
    y = torch.empty_like(x)
    B.layernorm(x, g, b, y)
    ref = torch.nn.functional.layer_norm(x.float(), (200,), g.float(), b.float())
    assert (y.float() - ref).abs().max().item() < 5e-2
    dy = torch.randn_like(x)
    dx = torch.empty_like(x)
    dg = torch.empty(200, device="cuda")
    db = torch.empty(200, device="cuda")
    B.layernorm_backward(x, g, dy, dx, dg, db)
    s = torch.randn(4, 50, 64, device="cuda").bfloat16()
    p = torch.empty_like(s)
    B.softmax(s, p)
    assert (p.float() - torch.softmax(s.float(), -1)).abs().max().item() < 1e-2
    B.masked_softmax(s, p, alpha=0.125)
    m = (torch.rand(4, 50, 64, device="cuda") < 0.3).to(torch.uint8)  # streamed + TMA stores
    B.masked_softmax(s, p, 0.125, m, -1e4)
    ref = torch.softmax(0.125 * s.float() - 1e4 * m.float(), -1)
    assert (p.float() - ref).abs().max().item() < 1e-2
    # general transpose (row-copy and tile kernels) and softmax over a middle axis
    for perm in ((1, 0, 2), (2, 0, 1)):
        q = torch.empty(tuple(s.shape[i] for i in perm), device="cuda").bfloat16()
        B.permute(s, q, perm)
        assert torch.equal(q, s.permute(perm))
    sa = torch.empty_like(s)
    B.softmax_axis(s, sa, 1)
    assert (sa.float() - torch.softmax(s.float(), 1)).abs().max().item() < 1e-2
    dsa = torch.empty_like(s)
    B.softmax_axis_backward(sa, torch.randn_like(s), dsa, 1)
    ds = torch.empty_like(s)
    B.softmax_backward(p, torch.randn_like(s), ds, alpha=0.125)
    t = torch.empty(4, 64, 50, device="cuda").bfloat16()
    B.transpose_last2(s, t)
    assert torch.equal(t, s.transpose(1, 2))
    ids = torch.randint(0, 97, (300,), device="cuda")
    table = torch.randn(97, 64, device="cuda").bfloat16()
    e = torch.empty(300, 64, device="cuda").bfloat16()
    B.embedding(ids, table, e)
    assert torch.equal(e, table[ids])
    dt = torch.zeros(97, 64, device="cuda")
    B.embedding_backward(ids, torch.randn(300, 64, device="cuda").bfloat16(), dt)
    torch.cuda.synchronize()


def peer():
    from oracle import data as O
    from paper_2302_02599_b200 import _capi as A
    from paper_2302_02599_b200 import DeviceMesh, ShardingSpec, TensorMeta
    from paper_2302_02599_b200.layout import check

    P = 4
    lib = A.lib()
    geo = DeviceMesh.uniform([2, 2])
    meshes = []
    for r in range(P):
        h = C.c_void_p()
        check(lib.apl_mesh_create_peer(C.byref(geo.c()), r, 0, C.byref(h)))
        meshes.append(h)
    streams = [torch.cuda.Stream() for _ in range(P)]
    flags = [torch.zeros(2 * P, dtype=torch.int32, device="cuda") for _ in range(P)]
    counters = [torch.zeros(4, dtype=torch.int32, device="cuda") for _ in range(P)]
    all_flags = (C.c_void_p * P)(*[f.data_ptr() for f in flags])
    epoch = 0
    for shape, a, b in [((64, 48), "S0S1", "S1S0"), ((64, 40), "S01R", "RS01"),
                        ((32, 32), "RR", "S0S1")]:
        meta = TensorMeta(shape, 2)
        s, t = ShardingSpec.parse(a, 2), ShardingSpec.parse(b, 2)
        g = O.fill_global(shape, 2)
        srcs = [torch.from_numpy(np.ascontiguousarray(x).view(np.int16)).cuda()
                for x in O.shards(g, O.parse_spec(a, 2), [2, 2])]
        want = O.shards(g, O.parse_spec(b, 2), [2, 2])
        table = (C.c_void_p * P)(*[x.data_ptr() for x in srcs])
        outs = [torch.empty(t.local_shape(meta, geo), dtype=torch.int16, device="cuda")
                for _ in range(P)]
        torch.cuda.synchronize()
        epoch += 1
        for r in range(P):
            sync = A.PeerSyncC(all_flags, flags[r].data_ptr(), counters[r].data_ptr(), epoch,
                               30000)
            check(lib.apl_run_pull_sync(meshes[r], C.byref(s.c()), C.byref(t.c()),
                                        C.byref(meta.c()), table, C.c_void_p(outs[r].data_ptr()),
                                        C.byref(sync), C.c_void_p(streams[r].cuda_stream)))
        torch.cuda.synchronize()
        for o, w in zip(outs, want):
            assert o.cpu().numpy().tobytes() == w.tobytes(), (a, b)
        # the push form: remote stores into every rank's output
        pouts = [torch.full(t.local_shape(meta, geo), -1, dtype=torch.int16, device="cuda")
                 for _ in range(P)]
        ptable = (C.c_void_p * P)(*[x.data_ptr() for x in pouts])
        torch.cuda.synchronize()
        epoch += 1
        for r in range(P):
            sync = A.PeerSyncC(all_flags, flags[r].data_ptr(), counters[r].data_ptr(), epoch,
                               30000)
            check(lib.apl_run_push_sync(meshes[r], C.byref(s.c()), C.byref(t.c()),
                                        C.byref(meta.c()), C.c_void_p(srcs[r].data_ptr()), ptable,
                                        C.byref(sync), C.c_void_p(streams[r].cuda_stream)))
        torch.cuda.synchronize()
        for o, w in zip(pouts, want):
            assert o.cpu().numpy().tobytes() == w.tobytes(), ("push", a, b)
    for h in meshes:
        lib.apl_mesh_destroy(h)


if __name__ == "__main__":
    torch.cuda.set_device(0)
    which = sys.argv[1:] or ["copies", "gemm", "block", "peer"]
    for w in which:
        globals()[w]()
        print(f"sanitize case {w}: ok", flush=True)
