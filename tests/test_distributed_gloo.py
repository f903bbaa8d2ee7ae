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
