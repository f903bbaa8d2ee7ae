"""Box-copy kernel sweep on one B200 (simulated meshes): GB/s of algorithmic
HBM bytes (source read once + destinations written) per conversion, next to
torch's own copy_ of the same bytes. One JSON line per conversion.

    APL_COPY_VARIANT=<v> python tools/copy_bench.py [--quick]
"""
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2302_02599_b200 import ShardingSpec, TensorMeta, find_transform_path  # noqa: E402
from paper_2302_02599_b200.runtime import Mesh  # noqa: E402

CASES = [
    # (mesh, shape, dtype_bytes, src, tgt)
    ([8], (65536, 8192), 2, "S0R", "S0R"),     # identity: pure 1 GiB copy
    ([8], (65536, 8192), 2, "S0R", "RR"),      # config 2 all-gather
    ([8], (65536, 8192), 2, "S0R", "RS0"),     # config 2 all-to-all
    ([8], (8192, 8192), 4, "S0R", "RS0"),
    ([2, 4], (8192, 8192), 2, "S01R", "S1S0"),  # config 3
    ([2, 4], (8192, 8192), 2, "S0S1", "RS01"),
    ([2, 4], (8192, 8192), 2, "RR", "S01R"),   # slice only
    ([2, 2, 2], (8192, 8192), 2, "S012R", "RS012"),  # config 4
    ([2, 2, 2], (512, 512, 256), 2, "S0S1R", "RS1S0"),
    ([2, 2, 2], (4096, 4096, 32), 2, "RS012R", "RRS012"),  # innermost-dim A2A (64 B runs)
    ([8], (1 << 21, 64), 2, "S0R", "RS0"),     # 16 B runs per receiver (split rows)
    ([8], (1 << 22, 32), 4, "S0R", "RS0"),     # 16 B runs, fp32
    ([2, 4], (1 << 20, 128), 2, "S01R", "RS01"),  # 32 B runs
]


def ev_time(fn, iters):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def sweep():
    """BASELINE config 2: mesh [8], S0R->RR and S0R->RS0, global 1 MiB .. 4 GiB,
    shape [T/(e*8192), 8192], fp32 and bf16 (collapsed exchange, one launch)."""
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] \
        if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
    mesh = Mesh.local([8])
    for eb, dt in ((4, torch.int32), (2, torch.int16)):
        for k in range(20, 33):
            total = 1 << k
            rows = total // (eb * 8192)
            if rows < 8:
                continue
            meta = TensorMeta((rows, 8192), eb)
            s = ShardingSpec.parse("S0R", 1)
            ins = [torch.randint(-100, 100, s.local_shape(meta, mesh.geo), dtype=dt, device="cuda")
                   for _ in range(8)]
            for tgt in ("RR", "RS0"):
                t = ShardingSpec.parse(tgt, 1)
                path = find_transform_path(s, t, mesh.geo, meta)
                outs = [torch.empty(t.local_shape(meta, mesh.geo), dtype=dt, device="cuda")
                        for _ in range(8)]
                tr = mesh.exchange_traffic(s, t, meta)
                nbytes = tr["hbm_read"] + tr["hbm_write"]
                iters = max(3, min(200, int(2e9 // max(nbytes, 1))))
                conv = mesh.prepare(path, meta, fuse=True)
                ms = ev_time(lambda: conv(ins, outs), iters)
                # device-side time: the same calls captured into one CUDA graph
                g = torch.cuda.CUDAGraph()
                side = torch.cuda.Stream()
                side.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(side):
                    conv(ins, outs, stream=side)
                    side.synchronize()
                    with torch.cuda.graph(g, stream=side):
                        for _ in range(10):
                            conv(ins, outs, stream=side)
                torch.cuda.current_stream().wait_stream(side)
                gms = ev_time(g.replay, max(3, iters // 10)) / 10
                print(json.dumps({"case": f"[8] S0R->{tgt}", "global_bytes": total, "eb": eb,
                                  "alg_bytes": nbytes, "ms": round(ms, 5),
                                  "gbs": round(nbytes / ms / 1e6, 1),
                                  "frac": round(nbytes / ms / 1e6 / peak, 3),
                                  "graph_ms": round(gms, 5),
                                  "graph_gbs": round(nbytes / gms / 1e6, 1),
                                  "graph_frac": round(nbytes / gms / 1e6 / peak, 3)}), flush=True)
                conv.close()
                del outs
            del ins
            torch.cuda.empty_cache()


def main():
    if "--sweep" in sys.argv:
        return sweep()
    quick = "--quick" in sys.argv
    variant = os.environ.get("APL_COPY_VARIANT", "0")
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] \
        if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
    x = torch.empty(1 << 29, dtype=torch.bfloat16, device="cuda")
    y = torch.empty_like(x)
    ms = ev_time(lambda: y.copy_(x), 10)
    print(json.dumps({"case": "torch copy_ 1 GiB", "variant": variant,
                      "gbs": round(2 * x.numel() * 2 / ms / 1e6, 1), "ms": round(ms, 4)}))
    del x, y
    for mesh_shape, shape, eb, a, b in (CASES[:3] if quick else CASES):
        mesh = Mesh.local(mesh_shape)
        mr = len(mesh_shape)
        meta = TensorMeta(shape, eb)
        s, t = ShardingSpec.parse(a, mr), ShardingSpec.parse(b, mr)
        path = find_transform_path(s, t, mesh.geo, meta)
        dt = {1: torch.uint8, 2: torch.int16, 4: torch.int32, 8: torch.int64}[eb]
        ins = [torch.randint(-100, 100, s.local_shape(meta, mesh.geo), dtype=dt, device="cuda")
               for _ in range(mesh.num_devices)]
        outs = [torch.empty(t.local_shape(meta, mesh.geo), dtype=dt, device="cuda")
                for _ in range(mesh.num_devices)]
        tr = mesh.exchange_traffic(s, t, meta)
        nbytes = tr["hbm_read"] + tr["hbm_write"]
        row = {"case": f"{mesh_shape} {list(shape)} e{eb} {a}->{b}", "variant": variant,
               "ref_steps": len(path.steps), "alg_bytes": nbytes}
        for fuse in (True, False):
            ms = ev_time(lambda: mesh.run_path(path, meta, ins, outs, fuse=fuse), 5 if quick else 20)
            key = "fused" if fuse else "stepwise"
            row[f"{key}_ms"] = round(ms, 4)
            row[f"{key}_gbs"] = round(nbytes / ms / 1e6, 1)
        row["fused_frac"] = round(row["fused_gbs"] / peak, 3)
        print(json.dumps(row), flush=True)
        del ins, outs, mesh
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
