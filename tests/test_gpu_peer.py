"""The fused peer-memory exchange on real hardware: one process per mesh
rank (4 and 8 ranks sharing cuda:0 through CUDA IPC), each rank pulling its
target shard out of the other ranks' exported source shards with ONE kernel
(apl_run_pull). Bytes must equal the CPU oracle on every rank. Handles and
barriers travel over gloo."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from test_gpu_nccl import drain

pytestmark = pytest.mark.gpu

CASES = {
    4: [([2, 2], (1024, 512), 2, "S0R", "RS0"), ([2, 2], (256, 384), 4, "S01R", "RS10"),
        ([2, 2], (64, 96, 32), 2, "S0S1R", "RS1S0"), ([4], (4096, 256), 2, "S0R", "RR"),
        ([2, 2], (128, 128), 1, "S1S0", "S0S1")],
    8: [([2, 4], (2048, 2048), 2, "S01R", "S1S0"), ([2, 4], (2048, 2048), 2, "S0S1", "RS01"),
        ([2, 4], (2048, 2048), 2, "RS01", "RR"), ([2, 2, 2], (2048, 2048), 2, "S012R", "RS012"),
        ([2, 2, 2], (128, 128, 64), 2, "S0S1R", "RS1S0"), ([8], (8192, 1024), 2, "S0R", "RS0")],
}


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cases, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from oracle import data as O
    from paper_2302_02599_b200 import ShardingSpec, TensorMeta
    from paper_2302_02599_b200.runtime import PeerMesh

    dt = {1: torch.uint8, 2: torch.int16, 4: torch.int32}
    try:
        biggest = max(int(np.prod(s)) * eb for _, s, eb, _, _ in cases)
        for mesh_shape, shape, eb, a, b in cases:
            pm = PeerMesh(mesh_shape, rank, 0, biggest)
            mr = len(mesh_shape)
            meta = TensorMeta(shape, eb)
            g = O.fill_global(shape, eb)
            mine = O.local(g, O.parse_spec(a, mr), mesh_shape, rank)
            want = O.local(g, O.parse_spec(b, mr), mesh_shape, rank)
            src = pm.shard(mine.shape, dt[eb])
            src.copy_(torch.from_numpy(mine.view(np.dtype(f"i{eb}") if eb > 1 else np.uint8)))
            out = torch.full(want.shape, -1, dtype=dt[eb], device="cuda:0")
            pm.exchange(ShardingSpec.parse(a, mr), ShardingSpec.parse(b, mr), meta, out)
            q.put((rank, a, b, out.cpu().numpy().tobytes() == want.tobytes()))
            pm.close()
            dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [4, 8])
def test_peer_pull_exchange_multiprocess(cuda, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, CASES[world], q))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    res = []
    while not q.empty():
        res.append(q.get())
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert len(res) == world * len(CASES[world])
    assert all(ok for *_, ok in res), [r for r in res if not r[-1]]


CONFIG3 = ["S01R", "S0S1", "S1S0", "RS01", "RR"]
FULL_CASES = (
    [([2, 4], (8192, 8192), 2, a, b) for a in CONFIG3 for b in CONFIG3 if a != b]
    + [([2, 2, 2], (8192, 8192), 2, "S012R", "RS012"), ([2, 2, 2], (8192, 8192), 2, "RS012", "S012R"),
       ([2, 2, 2], (512, 512, 256), 2, "S0S1R", "RS1S0"),
       ([2, 2, 2], (512, 512, 256), 2, "RS1S0", "S0S1R")])


def test_peer_pull_config3_config4_full_size(cuda):
    """BASELINE configs 3 and 4 at their named sizes on 8 ranks: all 20
    config-3 pairs on 2x4 ([8192, 8192] bf16) and the config-4 chains on
    2x2x2 ([8192, 8192] and [512, 512, 256]), one pull kernel per rank,
    bytewise vs the oracle on every rank."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 8, port, FULL_CASES, q)) for r in range(8)]
    for p in procs:
        p.start()
    res = drain(procs, q, 900)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert len(res) == 8 * len(FULL_CASES)
    assert all(ok for *_, ok in res), [r for r in res if not r[-1]]


EPOCH_CASES = {
    4: [([2, 2], (1024, 512), 2, "S0R", "RS0"), ([4], (2048, 256), 4, "S0R", "RR")],
    8: [([2, 4], (1024, 1024), 2, "S01R", "S1S0"), ([2, 2, 2], (1024, 512), 2, "S012R", "RS012")],
}
EPOCHS = 3


def _epoch_worker(rank, world, port, cases, q, fused=True):
    """Repeated exchanges synchronised only on the device: each epoch the
    rank rewrites its exported source (after wait_readers) with a different
    tensor, then exchange_async; no host barrier between epochs."""
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from oracle import data as O
    from paper_2302_02599_b200 import ShardingSpec, TensorMeta
    from paper_2302_02599_b200.runtime import PeerMesh

    dt = {1: torch.uint8, 2: torch.int16, 4: torch.int32}
    npdt = {1: np.uint8, 2: np.int16, 4: np.int32}
    try:
        for mesh_shape, shape, eb, a, b in cases:
            mr = len(mesh_shape)
            meta = TensorMeta(shape, eb)
            nbytes = int(np.prod(shape)) * eb
            pm = PeerMesh(mesh_shape, rank, 0, nbytes)
            srcs, wants = [], []
            for e in range(EPOCHS):  # stage every epoch's source on the device up front
                g = O.fill_global(shape, eb, seed=1000 + e)
                mine = O.local(g, O.parse_spec(a, mr), mesh_shape, rank)
                srcs.append(torch.from_numpy(mine.view(npdt[eb])).cuda())
                wants.append(O.local(g, O.parse_spec(b, mr), mesh_shape, rank))
            torch.cuda.synchronize()
            dist.barrier()  # setup only; the epochs below never meet on the host
            outs = []
            for e in range(EPOCHS):
                pm.wait_readers()
                pm.shard(srcs[e].shape, dt[eb]).copy_(srcs[e])
                out = torch.full(wants[e].shape, -1, dtype=dt[eb], device="cuda:0")
                pm.exchange_async(ShardingSpec.parse(a, mr), ShardingSpec.parse(b, mr), meta, out,
                                  fused=fused)
                outs.append(out)
            pm.wait_readers()
            torch.cuda.synchronize()
            for e in range(EPOCHS):
                q.put((rank, a, b, e, outs[e].cpu().numpy().tobytes() == wants[e].tobytes()))
            dist.barrier()
            pm.close()
            dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("world", [4, 8])
def test_peer_exchange_device_synchronised_epochs(cuda, world, fused):
    """fused: one launch per exchange (apl_run_pull_sync); unfused: flag
    store / flag wait / pull / flag store kernels."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_epoch_worker, args=(r, world, port, EPOCH_CASES[world], q, fused))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    res = []
    while not q.empty():
        res.append(q.get())
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert len(res) == world * len(EPOCH_CASES[world]) * EPOCHS
    assert all(ok for *_, ok in res), [r for r in res if not r[-1]]


def _allreduce_worker(rank, world, port, q):
    """Megatron fc2 (split-k over all ranks) with the GEMM and its all-reduce
    fused over peer memory, two epochs with fresh operands."""
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2302_02599_b200.runtime import PeerMesh

    try:
        M, Kt, N = 1024, 2048, 512
        kr = Kt // world
        pm = PeerMesh([world], rank, 0, 16)
        for epoch in range(2):
            g = torch.Generator(device="cuda").manual_seed(100 + epoch)
            x = torch.randn(M, Kt, device="cuda", generator=g).bfloat16()
            w = (torch.randn(Kt, N, device="cuda", generator=g) / Kt ** 0.5).bfloat16()
            a = x[:, rank * kr:(rank + 1) * kr].contiguous()
            b = w[rank * kr:(rank + 1) * kr].contiguous()
            for out_dtype in (torch.bfloat16, torch.float32):
                c = pm.matmul_allreduce(a, b, out_dtype=out_dtype)
                torch.cuda.synchronize()
                ref = x.double() @ w.double()
                err = ((c.double() - ref).abs().max() / ref.abs().max()).item()
                tol = 2e-2 if out_dtype == torch.bfloat16 else 1e-5
                digest = c.view(torch.uint8).sum(dtype=torch.int64).item()
                q.put((rank, epoch, str(out_dtype), err <= tol, err, digest))
        # config 5, Megatron selection through PeerMesh.sharded_matmul: fc1
        # split-n:0 (local GEMM + GELU), fc2 split-k:0 (fused GEMM + all-reduce)
        from paper_2302_02599_b200 import ShardingSpec
        from paper_2302_02599_b200.runtime import MatmulStrategy

        g = torch.Generator(device="cuda").manual_seed(7)
        x = torch.randn(1024, 256, device="cuda", generator=g).bfloat16()
        w1 = (torch.randn(256, 1024, device="cuda", generator=g) / 16).bfloat16()
        w2 = (torch.randn(1024, 256, device="cuda", generator=g) / 32).bfloat16()
        hs = 1024 // world
        p = lambda s: ShardingSpec.parse(s, 1)  # noqa: E731
        h = pm.sharded_matmul(MatmulStrategy("split-n:0", p("RR"), p("RS0"), p("RS0")), x,
                              w1[:, rank * hs:(rank + 1) * hs].contiguous(), gelu=True)
        y = pm.sharded_matmul(MatmulStrategy("split-k:0", p("RS0"), p("S0R"), p("RR"), [0]), h,
                              w2[rank * hs:(rank + 1) * hs].contiguous())
        torch.cuda.synchronize()
        ref = torch.nn.functional.gelu(x.double() @ w1.double()) @ w2.double()
        err = ((y.double() - ref).abs().max() / ref.abs().max()).item()
        q.put((rank, 9, "megatron", err <= 2e-2, err, y.view(torch.uint8).sum(dtype=torch.int64).item()))
        dist.barrier()
        pm.close()
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [4, 8])
def test_fused_gemm_allreduce_over_peer_memory(cuda, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_allreduce_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    res = []
    while not q.empty():
        res.append(q.get())
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert len(res) == world * 5
    assert all(r[3] for r in res), [r for r in res if not r[3]]
    assert len({r[5] for r in res if r[2] == "megatron"}) == 1
    for epoch in range(2):  # every rank holds the same bytes
        for dt in ("torch.bfloat16", "torch.float32"):
            assert len({r[5] for r in res if r[1] == epoch and r[2] == dt}) == 1


def _subset_allreduce_worker(rank, world, port, q):
    """Fused GEMM + all-reduce over a SUBSET of a 2-D peer mesh's axes (the
    reference's split-k strategies on one axis of a 2-D mesh, e.g. reduce_axes
    (1,) of split-mk:0,1): each reduce group sums only its own members'
    partials, groups run independently on different operands; then GELU after
    the sum through PeerMesh.sharded_matmul."""
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2302_02599_b200 import ShardingSpec
    from paper_2302_02599_b200.runtime import MatmulStrategy, PeerMesh

    try:
        shape = [2, world // 2]
        pm = PeerMesh(shape, rank, 0, 16)
        coord = (rank // shape[1], rank % shape[1])
        # M / group size must be whole 128-row tiles for the fused scatter
        M, Kt, N = 128 * world, 1024, 256
        for axes in ((0,), (1,), (0, 1)):
            members = pm.axis_group(axes)
            me, P = members.index(rank), len(members)
            # the operands of this rank's group: seeded by the coordinates off `axes`
            key = sum(c * 10 ** i for i, c in enumerate(coord) if i not in axes)
            g = torch.Generator(device="cuda").manual_seed(500 + key)
            x = torch.randn(M, Kt, device="cuda", generator=g).bfloat16()
            w = (torch.randn(Kt, N, device="cuda", generator=g) / Kt ** 0.5).bfloat16()
            kr = Kt // P
            a = x[:, me * kr:(me + 1) * kr].contiguous()
            b = w[me * kr:(me + 1) * kr].contiguous()
            c = pm.matmul_allreduce(a, b, out_dtype=torch.float32, axes=axes)
            torch.cuda.synchronize()
            ref = x.double() @ w.double()
            err = ((c.double() - ref).abs().max() / ref.abs().max()).item()
            q.put((rank, str(axes), err <= 1e-5, err, key, c.view(torch.uint8).sum(dtype=torch.int64).item()))
            st = MatmulStrategy("split-k", ShardingSpec.parse("RR", 2), ShardingSpec.parse("RR", 2),
                                ShardingSpec.parse("RR", 2), list(axes))
            h = pm.sharded_matmul(st, a, b, gelu=True)
            torch.cuda.synchronize()
            ref = torch.nn.functional.gelu(ref)
            err = ((h.double() - ref).abs().max() / ref.abs().max()).item()
            q.put((rank, str(axes) + "+gelu", err <= 2e-2, err, key, 0))
        dist.barrier()
        pm.close()
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [4, 8])
def test_fused_gemm_allreduce_over_axis_subsets(cuda, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_subset_allreduce_worker, args=(r, world, port, q))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    res = []
    while not q.empty():
        res.append(q.get())
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert len(res) == world * 6
    assert all(r[2] for r in res), [r for r in res if not r[2]]
    for axes in ("(0,)", "(1,)", "(0, 1)"):  # replicas inside a group: identical bytes
        by_group = {}
        for r in res:
            if r[1] == axes:
                by_group.setdefault(r[4], set()).add(r[5])
        assert all(len(v) == 1 for v in by_group.values()), (axes, by_group)


def _push_worker(rank, world, port, cases, q):
    """Push exchanges (remote stores into the receivers' exported outputs),
    synchronised only on the device, several epochs back to back with a
    different source each epoch; every output checked against the oracle."""
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from oracle import data as O
    from paper_2302_02599_b200 import ShardingSpec, TensorMeta
    from paper_2302_02599_b200.runtime import PeerMesh

    dt = {1: torch.uint8, 2: torch.int16, 4: torch.int32}
    npdt = {1: np.uint8, 2: np.int16, 4: np.int32}
    try:
        for mesh_shape, shape, eb, a, b in cases:
            mr = len(mesh_shape)
            meta = TensorMeta(shape, eb)
            pm = PeerMesh(mesh_shape, rank, 0, 16)
            s, t = ShardingSpec.parse(a, mr), ShardingSpec.parse(b, mr)
            pm.push_output(t.per_device_bytes(meta, pm.geo))  # collective allocation
            srcs, wants = [], []
            for e in range(EPOCHS):
                g = O.fill_global(shape, eb, seed=2000 + e)
                srcs.append(torch.from_numpy(O.local(g, O.parse_spec(a, mr), mesh_shape, rank)
                                             .view(npdt[eb])).cuda())
                wants.append(O.local(g, O.parse_spec(b, mr), mesh_shape, rank))
            torch.cuda.synchronize()
            dist.barrier()  # setup only
            outs = []
            for e in range(EPOCHS):
                out = pm.push_async(s, t, meta, srcs[e])
                outs.append(out.view(dt[eb]).clone())  # consume before the next epoch
            torch.cuda.synchronize()
            for e in range(EPOCHS):
                q.put((rank, a, b, e, outs[e].cpu().numpy().tobytes() == wants[e].tobytes()))
            dist.barrier()
            pm.close()
            dist.barrier()
    finally:
        dist.destroy_process_group()


PUSH_CASES = {
    4: EPOCH_CASES[4] + [([2, 2], (512, 256), 2, "RR", "S01R"), ([4], (64, 32), 2, "RS0", "S0R")],
    8: EPOCH_CASES[8] + [([8], (2048, 256), 2, "S0R", "RR"), ([2, 4], (512, 512), 2, "S0S1", "RS01")],
}


@pytest.mark.parametrize("world", [4, 8])
def test_peer_push_exchange_epochs(cuda, world):
    """apl_run_push_sync: the push form of the peer exchange (remote stores,
    fan-out descriptors for replicated targets) against the oracle."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_push_worker, args=(r, world, port, PUSH_CASES[world], q))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    res = []
    while not q.empty():
        res.append(q.get())
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert len(res) == world * len(PUSH_CASES[world]) * EPOCHS
    assert all(ok for *_, ok in res), [r for r in res if not r[-1]]
