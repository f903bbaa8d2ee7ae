"""Peer-exchange latency: one fused launch per exchange vs the 4-launch form
(flag store, flag wait, pull, flag store). N ranks (torchrun), each on
LOCAL_RANK % device_count (so N ranks may share one GPU: then kernels of
different processes time-slice and the numbers include that).

    python -m torch.distributed.run --nproc-per-node 8 tools/peer_latency.py

Prints one JSON line per case (rank 0): us per exchange (max over ranks of
the event time over `iters` back-to-back exchanges with wait_readers before
each), launches per exchange, bytes pulled per rank.
"""
import argparse
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2302_02599_b200 import ShardingSpec, TensorMeta  # noqa: E402
from paper_2302_02599_b200.runtime import PeerMesh, launch_count  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=50)
    args = ap.parse_args()
    ws, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    dev = int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")
    cases = [("tiny", (8 * ws, 256), "S0R", "RS0"),          # 4 KiB shards
             ("16MiB-AG", (1024 * ws, 1024), "S0R", "RR"),    # 2 MiB shard -> 16 MiB at N=8
             ("16MiB-A2A", (8192 * ws, 1024), "S0R", "RS0")]  # 16 MiB shard per rank
    for name, shape, a, b in cases:
        meta = TensorMeta(shape, 2)
        s, t = ShardingSpec.parse(a, 1), ShardingSpec.parse(b, 1)
        pm = PeerMesh([ws], rank, dev, shape[0] // ws * shape[1] * 2)
        src = pm.shard(s.local_shape(meta, pm.geo), torch.bfloat16)
        src.view(torch.int16).random_(-100, 100)
        out = torch.empty(t.local_shape(meta, pm.geo), dtype=torch.bfloat16, device=f"cuda:{dev}")
        wire = pm.exchange_traffic(s, t, meta)["wire_in"]
        stream = torch.cuda.current_stream()
        row = {"case": name, "ranks": ws, "tensor": list(shape), "conversion": f"{a}->{b}",
               "bytes_pulled_per_rank": wire,
               "gpus_shared": torch.cuda.device_count() < ws}
        for fused in (True, False):
            for _ in range(5):
                pm.wait_readers(stream=stream)
                pm.exchange_async(s, t, meta, out, stream=stream, fused=fused)
            torch.cuda.synchronize()
            dist.barrier()
            l0 = launch_count()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.iters):
                pm.wait_readers(stream=stream)
                pm.exchange_async(s, t, meta, out, stream=stream, fused=fused)
            e1.record(stream)
            torch.cuda.synchronize()
            launches = (launch_count() - l0) / args.iters
            v = torch.tensor([e0.elapsed_time(e1) / args.iters * 1e3], dtype=torch.float64)
            dist.all_reduce(v, op=dist.ReduceOp.MAX)
            key = "fused" if fused else "unfused"
            row[f"{key}_us"] = round(float(v[0]), 2)
            row[f"{key}_launches_per_exchange"] = launches
            dist.barrier()
        pm.close()
        if rank == 0:
            print(json.dumps(row), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
