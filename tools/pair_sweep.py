"""Every spec-to-spec conversion of a mesh, timed: the north star's "every
conversion on a 2x4 and 2x2x2 mesh" at >= 64 MB, as pack HBM GB/s on one
B200 (simulated mesh; collapsed exchange through prepared conversions, the
public API). Specs are enumerated like the reference's enumerate_specs
(layout.cpp: every assignment of each mesh axis to at most one tensor dim,
in every order), pairs the reference path search accepts.

    python tools/pair_sweep.py [--mesh 2,4] [--shape 8192,8192] [--sample N] [--iters 10]

One JSON line per pair ({src, tgt, ref_steps, us, hbm_bytes, frac}), then a
summary line (min / p10 / median / max of frac, the slowest pairs).
"""
import argparse
import itertools
import json
import random
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2302_02599_b200 import ShardingSpec, TensorMeta, find_transform_path  # noqa: E402
from paper_2302_02599_b200.runtime import Mesh  # noqa: E402


def specs(rank, mesh_rank, shape, mesh_shape):
    """All valid specs: each mesh axis on at most one dim, ordered within a dim;
    every sharded dim divisible by its axes' product."""
    out = set()
    axes = list(range(mesh_rank))
    for assign in itertools.product(range(rank + 1), repeat=mesh_rank):  # rank = unassigned
        per_dim = [[a for a in axes if assign[a] == d] for d in range(rank)]
        for orders in itertools.product(*[list(itertools.permutations(p)) for p in per_dim]):
            ok = True
            for d, o in enumerate(orders):
                n = 1
                for a in o:
                    n *= mesh_shape[a]
                ok &= shape[d] % n == 0
            if ok:
                out.add("".join("R" if not o else "S" + "".join(map(str, o)) for o in orders))
    return sorted(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mesh", default="2,4")
    ap.add_argument("--shape", default="8192,8192")
    ap.add_argument("--sample", type=int, default=0, help="random subset of pairs (0: all)")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--peak", type=float, default=0.0)
    args = ap.parse_args()
    ms = [int(x) for x in args.mesh.split(",")]
    shape = tuple(int(x) for x in args.shape.split(","))
    peak = args.peak
    if not peak:
        p = ROOT / "MEASURED_PEAKS.json"
        peak = float(json.loads(p.read_text()).get("hbm_copy_gbs", 6457.1)) if p.exists() else 6457.1
    mesh = Mesh.local(ms)
    meta = TensorMeta(shape, 2)
    sp = specs(len(shape), len(ms), shape, ms)
    pairs = [(a, b) for a in sp for b in sp if a != b]
    if args.sample and args.sample < len(pairs):
        random.Random(2302).shuffle(pairs)
        pairs = pairs[:args.sample]
    stream = torch.cuda.current_stream()
    rows = []
    cache_in = {}
    for a, b in pairs:
        s, t = ShardingSpec.parse(a, len(ms)), ShardingSpec.parse(b, len(ms))
        path = find_transform_path(s, t, mesh.geo, meta)
        if a not in cache_in:
            cache_in.clear()
            cache_in[a] = [torch.empty(s.local_shape(meta, mesh.geo), dtype=torch.bfloat16,
                                       device="cuda").view(torch.int16).random_(-3000, 3000)
                           .view(torch.bfloat16) for _ in range(mesh.num_local)]
        ins = cache_in[a]
        outs = [torch.empty(t.local_shape(meta, mesh.geo), dtype=torch.bfloat16, device="cuda")
                for _ in range(mesh.num_local)]
        conv = mesh.prepare(path, meta, fuse=True)
        tr = mesh.exchange_traffic(s, t, meta)
        nbytes = tr["hbm_read"] + tr["hbm_write"]
        for _ in range(3):
            conv(ins, outs, stream=stream)
        torch.cuda.synchronize()
        ms_ = 1e30
        for _ in range(2):  # best of two rounds: a sporadic stall on the box is not the kernel
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.iters):
                conv(ins, outs, stream=stream)
            e1.record(stream)
            torch.cuda.synchronize()
            ms_ = min(ms_, e0.elapsed_time(e1) / args.iters)
        conv.close()
        row = {"src": a, "tgt": b, "ref_steps": len(path.steps), "us": round(ms_ * 1e3, 2),
               "hbm_bytes": nbytes, "frac": round(nbytes / (ms_ * 1e-3) / 1e9 / peak, 4)}
        rows.append(row)
        print(json.dumps(row), flush=True)
    fr = sorted(r["frac"] for r in rows)
    q = lambda p: fr[min(len(fr) - 1, int(p * len(fr)))]  # noqa: E731
    worst = sorted(rows, key=lambda r: r["frac"])[:10]
    print(json.dumps({"summary": True, "mesh": ms, "tensor": list(shape), "pairs": len(rows),
                      "specs": len(sp), "frac_min": fr[0], "frac_p10": q(0.1),
                      "frac_median": q(0.5), "frac_max": fr[-1], "peak_gbs": peak,
                      "worst": [(r["src"], r["tgt"], r["frac"]) for r in worst]}), flush=True)
    mesh.close()


if __name__ == "__main__":
    main()
