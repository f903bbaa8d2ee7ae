"""The NCCL transport executed for real: 2, 4 and 8 ranks on cuda:0.

NCCL refuses two ranks of one host on the same GPU ("Duplicate GPU
detected"), so every rank gets its own NCCL_HOSTID: NCCL then treats the
ranks as separate hosts and connects them over its socket transport on the
loopback interface. The data plane is the production one -- ncclAllGather /
ncclAlltoAll on the mesh-axis communicators (ncclCommSplit per axis subset),
grouped ncclSend/ncclRecv for collapsed chains, ncclAllReduce for partial
sums, plus this library's pack/unpack kernels -- only the wire is slower
than NVLink. Every rank's bytes must equal the CPU oracle (reference step
semantics: planner.cpp:263-347 insertion points, cluster.hpp:46-52
collective vocabulary)."""
import os
import queue
import socket
import time

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

CONFIG3 = ["S01R", "S0S1", "S1S0", "RS01", "RR"]

# (mesh, [(shape, eb, src, tgt)]) per world size
CASES = {
    2: [([2], [((1024, 512), 2, "S0R", "RR"), ((1024, 512), 2, "S0R", "RS0"),
               ((1024, 512), 2, "RS0", "S0R"), ((256, 384), 4, "RS0", "RR"),
               ((64, 96, 32), 4, "S0RR", "RRS0"), ((64, 96, 32), 1, "RRS0", "RS0R"),
               ((512, 512), 2, "RR", "S0R"), ((2, 8), 8, "S0R", "RS0")])],
    4: [([2, 2], [((1024, 1024), 4, "S0R", "RS0"), ((1024, 1024), 2, "S01R", "RS01"),
                  ((1024, 1024), 2, "S0S1", "S1S0"), ((1024, 1024), 2, "RR", "S01R"),
                  ((1024, 1024), 2, "S01R", "RR"), ((64, 96, 32), 2, "S0S1R", "RS1S0"),
                  ((256, 128), 1, "S10R", "RS01")]),
        ([4], [((2048, 256), 2, "S0R", "RS0"), ((2048, 256), 4, "S0R", "RR")])],
    8: [([2, 4], [((512, 512), 2, a, b) for a in CONFIG3 for b in CONFIG3 if a != b]),
        ([2, 2, 2], [((512, 512), 2, "S012R", "RS012"), ((512, 512), 2, "RS012", "S012R"),
                     ((64, 64, 32), 2, "S0S1R", "RS1S0"), ((64, 64, 32), 2, "RS1S0", "S0S1R")]),
        ([8], [((8192, 256), 2, "S0R", "RR"), ((8192, 256), 2, "S0R", "RS0")])],
}


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def drain(procs, q, timeout):
    """Collect results while the workers run (a full result pipe must not
    block a worker's exit), then reap them."""
    res, deadline = [], time.monotonic() + timeout
    while any(p.is_alive() for p in procs) and time.monotonic() < deadline:
        try:
            res.append(q.get(timeout=0.2))
        except queue.Empty:
            pass
    while True:
        try:
            res.append(q.get(timeout=0.5))
        except queue.Empty:
            break
    for p in procs:
        if p.is_alive():
            p.kill()
        p.join()
    return res


def _worker(rank, world, port, cases, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                      NCCL_HOSTID=f"apl-nccl-test-host-{rank}", NCCL_SOCKET_IFNAME="lo",
                      NCCL_IB_DISABLE="1")
    import torch
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from oracle import data as O
    from paper_2302_02599_b200 import ShardingSpec, TensorMeta, find_transform_path
    from paper_2302_02599_b200.runtime import Mesh, launch_count

    dt = {1: torch.uint8, 2: torch.int16, 4: torch.int32, 8: torch.int64}
    npdt = {1: np.uint8, 2: np.int16, 4: np.int32, 8: np.int64}
    try:
        for mesh_shape, convs in cases:
            mesh = Mesh.from_process_group(mesh_shape)
            mr = len(mesh_shape)
            stream = torch.cuda.current_stream()
            for shape, eb, a, b in convs:
                meta = TensorMeta(shape, eb)
                s, t = ShardingSpec.parse(a, mr), ShardingSpec.parse(b, mr)
                path = find_transform_path(s, t, mesh.geo, meta)
                g = O.fill_global(shape, eb)
                mine = O.local(g, O.parse_spec(a, mr), mesh_shape, rank)
                want = O.local(g, O.parse_spec(b, mr), mesh_shape, rank)
                src = torch.from_numpy(mine.view(npdt[eb])).cuda()
                for mode in ("stepwise", "collapsed", "prepared"):
                    out = torch.full(want.shape, -1, dtype=dt[eb], device="cuda:0")
                    before = launch_count()
                    if mode == "prepared":
                        conv = mesh.prepare(path, meta, fuse=True)
                        conv([src], [out], stream=stream)
                        conv([src], [out], stream=stream)  # replay reuses the compiled exchange
                    else:
                        mesh.run_path(path, meta, [src], [out], fuse=mode == "collapsed",
                                      stream=stream)
                    mesh.synchronize(stream, timeout_s=120)
                    ok = out.cpu().numpy().view(want.dtype).tobytes() == want.tobytes()
                    q.put(("conv", rank, str(mesh_shape), f"{a}->{b}", mode, len(path.steps),
                           launch_count() - before, ok))
                    if mode == "prepared":
                        conv.close()
                dist.barrier()
            # partial-sum all-reduce on every axis subset (ncclAllReduce on the
            # subset communicator); each rank regenerates every member's part
            for mask in range(1, 1 << mr):
                axes = [x for x in range(mr) if mask >> x & 1]
                parts = [np.random.default_rng(100 * d + mask).standard_normal(4099)
                         .astype(np.float32) for d in range(mesh.geo.num_devices())]
                me = mesh.geo.coord_of(rank)
                group = [d for d in range(mesh.geo.num_devices())
                         if all(mesh.geo.coord_of(d)[x] == me[x] for x in range(mr)
                                if x not in axes)]
                want = np.sum(np.stack([parts[d].astype(np.float64) for d in group]), axis=0)
                buf = torch.from_numpy(parts[rank]).cuda()
                mesh.all_reduce(axes, [buf], stream=stream)
                mesh.synchronize(stream, timeout_s=120)
                err = float(np.max(np.abs(buf.cpu().numpy() - want)) / np.max(np.abs(want)))
                q.put(("ar", rank, str(mesh_shape), str(axes), "", 0, 0, err <= 1e-6))
            assert mesh.health() == 0
            dist.barrier()
            mesh.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_nccl_transport_multiprocess(cuda, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, CASES[world], q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = drain(procs, q, 900)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    n_conv = sum(len(c) for _, c in CASES[world]) * 3
    n_ar = sum((1 << len(m)) - 1 for m, _ in CASES[world])
    assert len([r for r in res if r[0] == "conv"]) == world * n_conv
    assert len([r for r in res if r[0] == "ar"]) == world * n_ar
    bad = [r for r in res if not r[-1]]
    assert not bad, bad[:10]
