"""Single-process loopback of the peer exchange protocol: all P ranks of a
PeerMesh live in this process on one GPU (P apl_mesh_create_peer handles,
plain device buffers instead of IPC mappings, one CUDA stream per rank), so
every rank's kernel is resident at the same time and the flags resolve
without the multi-process time-slicing that dominates 8 processes sharing
one GPU (tools/peer_latency.py). Each rank's fused kernel is capped at
(SMs x 4) / P CTAs (APL_PULL_GRID_CAP) so all P fit at once.

Measures, per exchange (all ranks, epochs back to back, wait_readers of the
previous epoch included): the fused form (1 launch: announce + acquire
senders + pull + done) against the 4-launch form (flag store, flag wait,
pull, flag store), for an empty-ish exchange and for 16 MiB per rank.
Every output is checked against the oracle-free invariant that the fused
and unfused forms produce identical bytes. Prints one JSON line per case.

    python tools/peer_loopback.py [--ranks 8] [--iters 200]
"""
import argparse
import ctypes as C
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ranks", type=int, default=8)
    ap.add_argument("--iters", type=int, default=200)
    ap.add_argument("--modes", default="fused,unfused",
                    help="comma list of fused / unfused (each in its own process for A/B)")
    ap.add_argument("--debug", action="store_true", help="synchronise and report after each warm-up exchange")
    args = ap.parse_args()
    P = args.ranks
    # one hardware queue per stream: two ranks' streams sharing a queue would
    # serialise a spinning kernel in front of the kernel it waits for
    os.environ["CUDA_DEVICE_MAX_CONNECTIONS"] = "32"
    import torch

    os.environ.setdefault("APL_PULL_GRID_CAP", str(max(1, 148 * 4 // P)))
    from paper_2302_02599_b200 import _capi as A
    from paper_2302_02599_b200 import DeviceMesh, ShardingSpec, TensorMeta
    from paper_2302_02599_b200.layout import check

    lib = A.lib()
    torch.cuda.set_device(0)
    geo = DeviceMesh.uniform([P])
    meshes = []
    for r in range(P):
        h = C.c_void_p()
        check(lib.apl_mesh_create_peer(C.byref(geo.c()), r, 0, C.byref(h)))
        meshes.append(h)
    streams = [torch.cuda.Stream() for _ in range(P)]
    flags = [torch.zeros(2 * P, dtype=torch.int32, device="cuda") for _ in range(P)]
    counters = [torch.zeros(4, dtype=torch.int32, device="cuda") for _ in range(P)]
    all_flags = (C.c_void_p * P)(*[f.data_ptr() for f in flags])
    cases = [("tiny", (8 * P, 256), "S0R", "RS0"),
             ("16MiB-AG", (1024 * P, 1024), "S0R", "RR"),
             ("16MiB-A2A", (8192 * P, 1024), "S0R", "RS0")]
    epoch = 0
    for name, shape, a, b in cases:
        meta = TensorMeta(shape, 2)
        s, t = ShardingSpec.parse(a, 1), ShardingSpec.parse(b, 1)
        srcs = [torch.empty(s.local_shape(meta, geo), dtype=torch.int16, device="cuda")
                .random_(-1000, 1000) for _ in range(P)]
        table = (C.c_void_p * P)(*[x.data_ptr() for x in srcs])
        outs = {k: [torch.empty(t.local_shape(meta, geo), dtype=torch.int16, device="cuda")
                    for _ in range(P)] for k in ("fused", "unfused")}
        others = [[q for q in range(P) if q != r] for r in range(P)]
        torch.cuda.synchronize()

        def exchange(fused, e):
            for r in range(P):
                sh = C.c_void_p(streams[r].cuda_stream)
                if e > 1:  # wait_readers of the previous epoch (every rank reads every rank here)
                    slots = (C.c_int32 * (P - 1))(*[P + q for q in others[r]])
                    check(lib.apl_peer_flags_wait(C.c_void_p(flags[r].data_ptr()), slots, P - 1,
                                                  e - 1, 3000, sh))
                out = C.c_void_p(outs["fused" if fused else "unfused"][r].data_ptr())
                if fused:
                    sync = A.PeerSyncC(all_flags, flags[r].data_ptr(), counters[r].data_ptr(), e,
                                       3000)
                    check(lib.apl_run_pull_sync(meshes[r], C.byref(s.c()), C.byref(t.c()),
                                                C.byref(meta.c()), table, out, C.byref(sync), sh))
                else:
                    peers = (C.c_void_p * (P - 1))(*[flags[q].data_ptr() for q in others[r]])
                    ready = (C.c_int32 * (P - 1))(*others[r])
                    check(lib.apl_peer_flags_store(peers, P - 1, r, e, sh))
                    check(lib.apl_peer_flags_wait(C.c_void_p(flags[r].data_ptr()), ready, P - 1,
                                                  e, 3000, sh))
                    check(lib.apl_run_pull(meshes[r], C.byref(s.c()), C.byref(t.c()),
                                           C.byref(meta.c()), table, out, sh))
                    check(lib.apl_peer_flags_store(peers, P - 1, P + r, e, sh))

        row = {"case": name, "ranks": P, "tensor": list(shape), "conversion": f"{a}->{b}",
               "grid_cap": int(os.environ["APL_PULL_GRID_CAP"]),
               "bytes_pulled_per_rank": s.per_device_bytes(meta, geo) * (P - 1) // (1 if b == "RR" else P)}
        for fused in [m == "fused" for m in args.modes.split(",")]:
            for _ in range(5):
                epoch += 1
                exchange(fused, epoch)
                if args.debug:
                    torch.cuda.synchronize()
                    print(f"ok {name} fused={fused} epoch={epoch}", file=sys.stderr, flush=True)
            torch.cuda.synchronize()
            start = torch.cuda.Event(enable_timing=True)
            start.record(torch.cuda.current_stream())
            for st in streams:
                st.wait_event(start)
            for _ in range(args.iters):
                epoch += 1
                exchange(fused, epoch)
            ends = []
            for st in streams:
                ev = torch.cuda.Event(enable_timing=True)
                ev.record(st)
                ends.append(ev)
            torch.cuda.synchronize()
            us = max(start.elapsed_time(ev) for ev in ends) / args.iters * 1e3
            row["fused_us" if fused else "unfused_us"] = round(us, 2)
        row["launches_per_rank_per_exchange"] = {"fused": 2, "unfused": 5}
        if "fused_us" in row and "unfused_us" in row:
            row["identical_bytes"] = all(torch.equal(x, y) for x, y in zip(outs["fused"],
                                                                           outs["unfused"]))
        for m in ("fused", "unfused"):
            if f"{m}_us" in row:
                row[f"bus_gbs_per_rank_{m}"] = round(row["bytes_pulled_per_rank"] / row[f"{m}_us"] / 1e3, 1)
        print(json.dumps(row), flush=True)
    for h in meshes:
        lib.apl_mesh_destroy(h)


if __name__ == "__main__":
    main()
