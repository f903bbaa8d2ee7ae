"""N>1 path on CPU: one process per mesh device over torch.distributed
(gloo, world size 4 and 8), each rank executing the EXACT schedule the
distributed (NCCL) executor compiles for it — pack/self copies, point-to-
point sends/recvs with their staging offsets, unpack copies — obtained from
libapl.so's host-only dry run (apl_exchange_schedule_json). Copies are
emulated with numpy (this file is test code); the result on every rank must
equal the CPU oracle bytewise."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

CASES = {
    4: [([2, 2], (64, 48), 4, "S0R", "RS0"), ([2, 2], (64, 48), 2, "S01R", "RS10"),
        ([2, 2], (8, 12, 6), 4, "S0S1R", "RS1S0"), ([4], (64, 32), 2, "S0R", "RR"),
        ([4], (64, 32), 2, "RR", "RS0"), ([2, 2], (16, 16), 1, "S1S0", "S0S1")],
    8: [([2, 4], (64, 64), 2, "S01R", "S1S0"), ([2, 4], (64, 64), 2, "S0S1", "RS01"),
        ([2, 4], (64, 64), 2, "RS01", "RR"), ([2, 2, 2], (64, 64), 2, "S012R", "RS012"),
        ([2, 2, 2], (16, 16, 8), 2, "S0S1R", "RS1S0"), ([8], (64, 128), 4, "S0R", "RS0")],
}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _copy(desc, srcs, dsts):
    """Emulates one CopyDesc of the box-copy kernel on byte buffers. A split
    descriptor (ksplit > 1) sends chunk j of every source row (src_off + j *
    split_src_step) to buffer split_dst[j] at split_dst_off[j]."""
    ext = tuple(desc["ext"]) + (desc["run_bytes"],)
    if desc.get("ksplit", 1) > 1:
        chunks = [(desc["src_off"] + j * desc["split_src_step"], b, off)
                  for j, (b, off) in enumerate(zip(desc["split_dst"], desc["split_dst_off"]))]
    else:
        chunks = [(desc["src_off"], desc["dst_buf"], desc["dst_off"])]
    src = srcs[desc["src_buf"]]
    for src_off, dst_buf, dst_off in chunks:
        sv = np.lib.stride_tricks.as_strided(src[src_off:], shape=ext,
                                             strides=tuple(desc["src_stride"]) + (1,))
        dv = np.lib.stride_tricks.as_strided(dsts[dst_buf][dst_off:], shape=ext,
                                             strides=tuple(desc["dst_stride"]) + (1,))
        dv[...] = sv


def _worker(rank, world, port, cases, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import data as O
    from paper_2302_02599_b200.layout import (DeviceMesh, ShardingSpec, TensorMeta,
                                              exchange_schedule)

    try:
        for mesh_shape, shape, eb, src, tgt in cases:
            mesh = DeviceMesh.uniform(mesh_shape)
            mr = len(mesh_shape)
            meta = TensorMeta(shape, eb)
            g = O.fill_global(shape, eb)
            mine = O.local(g, O.parse_spec(src, mr), mesh_shape, rank).view(np.uint8).ravel()
            want = O.local(g, O.parse_spec(tgt, mr), mesh_shape, rank).view(np.uint8).ravel()
            sch = exchange_schedule(mesh, rank, ShardingSpec.parse(src, mr),
                                    ShardingSpec.parse(tgt, mr), meta)
            out = np.full(want.size, 0xAB, dtype=np.uint8)
            send = np.zeros(max(1, sch["send_staging"]), dtype=np.uint8)
            recv = np.zeros(max(1, sch["recv_staging"]), dtype=np.uint8)
            for d in sch["pre"]:
                _copy(d, [mine, recv], [out, send])
            reqs, landing = [], []
            for peer, direct, off, n in sch["sends"]:
                buf = (mine if direct else send)[off:off + n]
                reqs.append(dist.isend(torch.from_numpy(buf.copy()), peer))
            for peer, direct, off, n in sch["recvs"]:
                t = torch.empty(n, dtype=torch.uint8)
                reqs.append(dist.irecv(t, peer))
                landing.append((direct, off, n, t))
            for r in reqs:
                r.wait()
            for direct, off, n, t in landing:
                (out if direct else recv)[off:off + n] = t.numpy()
            for d in sch["post"]:
                _copy(d, [mine, recv], [out, send])
            ok = out.tobytes() == want.tobytes()
            # a device never receives more than it lacks
            got = sum(n for _, _, _, n in sch["recvs"])
            q.put((rank, src, tgt, ok, got))
            dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [4, 8])
def test_distributed_schedule_over_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, CASES[world], q))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    results = []
    while not q.empty():
        results.append(q.get())
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert len(results) == world * len(CASES[world])
    bad = [r for r in results if not r[3]]
    assert not bad, bad


# Stepwise conversions on the distributed executor: every reference step is
# one hop -- an all-gather runs as ONE ncclAllGather and an all-to-all as ONE
# ncclAlltoAll on that mesh axis's communicator (emulated here with gloo on
# the axis group, members in coordinate order), a shard-slice as a local
# copy -- with intermediate shards between hops, exactly as
# apl_conversion_schedule_json reports for each rank.
STEP_CASES = {
    4: [([2, 2], (64, 48), 4, "S01R", "RR"), ([2, 2], (16, 8, 12), 2, "S0S1R", "RRS1"),
        ([4], (64, 32), 2, "S0R", "RR"), ([2, 2], (64, 48), 2, "S10R", "RS0"),
        ([4], (64, 32), 2, "S0R", "RS0"), ([2, 2], (8, 12, 16), 2, "S0S1R", "RS1S0"),
        ([2, 2], (16, 16), 1, "S1S0", "S0S1")],
    8: [([2, 4], (64, 64), 2, "S01R", "S1S0"), ([2, 2, 2], (64, 64), 2, "S012R", "RS012"),
        ([2, 4], (64, 64), 2, "RS01", "RR"), ([8], (64, 128), 4, "S0R", "RR"),
        ([8], (64, 128), 4, "S0R", "RS0"), ([2, 4], (64, 64), 2, "RS01", "S1S0")],
}


def _axis_groups(mesh_shape):
    """{axis: [ranks of each group]} -- devices differing only on the axis,
    ordered by their coordinate on it (the sub-communicator's rank order)."""
    import itertools

    r = len(mesh_shape)
    strides = [1] * r
    for i in range(r - 2, -1, -1):
        strides[i] = strides[i + 1] * mesh_shape[i + 1]
    out = {}
    for a in range(r):
        groups = []
        others = [range(n) if i != a else [0] for i, n in enumerate(mesh_shape)]
        for base in itertools.product(*others):
            groups.append([sum(c * s for c, s in zip(base, strides)) + j * strides[a]
                           for j in range(mesh_shape[a])])
        out[a] = groups
    return out


def _step_worker(rank, world, port, cases, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import data as O
    from paper_2302_02599_b200.layout import (DeviceMesh, ShardingSpec, TensorMeta,
                                              conversion_schedule, find_transform_path)

    try:
        for mesh_shape, shape, eb, src, tgt in cases:
            mesh = DeviceMesh.uniform(mesh_shape)
            mr = len(mesh_shape)
            meta = TensorMeta(shape, eb)
            # every rank creates every axis group in the same order (gloo rule)
            groups = {a: [(g, dist.new_group(g)) for g in gs]
                      for a, gs in _axis_groups(mesh_shape).items()}
            g = O.fill_global(shape, eb)
            cur = O.local(g, O.parse_spec(src, mr), mesh_shape, rank).view(np.uint8).ravel()
            want = O.local(g, O.parse_spec(tgt, mr), mesh_shape, rank).view(np.uint8).ravel()
            path = find_transform_path(ShardingSpec.parse(src, mr), ShardingSpec.parse(tgt, mr),
                                       mesh, meta)
            sch = conversion_schedule(mesh, rank, path, meta, fuse=False)
            n_ag = 0
            for hop in sch["hops"]:
                out = np.full(hop["out_bytes"], 0xAB, dtype=np.uint8)
                send = np.zeros(max(1, hop["send_staging"]), dtype=np.uint8)
                recv = np.zeros(max(1, hop["recv_staging"]), dtype=np.uint8)
                if "alltoall" in hop:
                    n_ag += 1
                    a2a = hop["alltoall"]
                    members, _ = next((m, gr) for m, gr in groups[a2a["axis"]] if rank in m)
                    ch = a2a["chunk"]
                    for d in hop["pre"]:
                        _copy(d, [cur, recv], [out, send])
                    sbuf = cur if a2a["direct_send"] else send
                    rbuf = out if a2a["direct_recv"] else recv
                    reqs, landing = [], []
                    for j, peer in enumerate(members):
                        if peer == rank:
                            me = members.index(rank)
                            rbuf[me * ch:(me + 1) * ch] = sbuf[me * ch:(me + 1) * ch]
                            continue
                        reqs.append(dist.isend(torch.from_numpy(sbuf[j * ch:(j + 1) * ch].copy()),
                                               peer))
                        t = torch.empty(ch, dtype=torch.uint8)
                        reqs.append(dist.irecv(t, peer))
                        landing.append((j, t))
                    for r in reqs:
                        r.wait()
                    for j, t in landing:
                        rbuf[j * ch:(j + 1) * ch] = t.numpy()
                    if not a2a["direct_recv"]:
                        for d in hop["post"]:
                            _copy(d, [cur, recv], [out, send])
                elif "allgather" in hop:
                    n_ag += 1
                    a = hop["allgather"]["axis"]
                    members, grp = next((m, gr) for m, gr in groups[a] if rank in m)
                    parts = [torch.empty(hop["in_bytes"], dtype=torch.uint8) for _ in members]
                    dist.all_gather(parts, torch.from_numpy(cur.copy()), group=grp)
                    gathered = torch.cat(parts).numpy()
                    if hop["allgather"]["direct"]:
                        out[:] = gathered
                    else:
                        recv[:gathered.size] = gathered
                        for d in hop["post"]:
                            _copy(d, [cur, recv], [out, send])
                else:
                    for d in hop["pre"]:
                        _copy(d, [cur, recv], [out, send])
                    reqs, landing = [], []
                    for peer, direct, off, n in hop["sends"]:
                        buf = (cur if direct else send)[off:off + n]
                        reqs.append(dist.isend(torch.from_numpy(buf.copy()), peer))
                    for peer, direct, off, n in hop["recvs"]:
                        t = torch.empty(n, dtype=torch.uint8)
                        reqs.append(dist.irecv(t, peer))
                        landing.append((direct, off, n, t))
                    for r in reqs:
                        r.wait()
                    for direct, off, n, t in landing:
                        (out if direct else recv)[off:off + n] = t.numpy()
                    for d in hop["post"]:
                        _copy(d, [cur, recv], [out, send])
                cur = out
                dist.barrier()
            q.put((rank, src, tgt, cur.tobytes() == want.tobytes(), n_ag))
            dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [4, 8])
def test_stepwise_schedule_with_axis_allgathers_over_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_step_worker, args=(r, world, port, STEP_CASES[world], q))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    results = []
    while not q.empty():
        results.append(q.get())
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert len(results) == world * len(STEP_CASES[world])
    bad = [r for r in results if not r[3]]
    assert not bad, bad
    assert all(r[4] >= 1 for r in results)  # the gathers / all-to-alls ran as collectives
