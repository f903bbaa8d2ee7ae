"""Size dependence of the copy engines on one B200 (simulated mesh [8]).

For each global size: torch copy_ of the same bytes (control), our identity
conversion (S0R->S0R: a plain copy through the box-copy machinery), the
all-to-all S0R->RS0, and the BASELINE config-3/4 conversions at 128 MiB.
Device time of 10 back-to-back calls captured in a CUDA graph.

    APL_COPY_ENGINE=ldg|bulk python tools/size_probe.py [--quick | --small]
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


def graph_ms(fn, reps=10, iters=5):
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        fn(side)
        side.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            for _ in range(reps):
                fn(side)
    torch.cuda.current_stream().wait_stream(side)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / (iters * reps)


def carve(n, shape, dt, skew):
    """n tensors of `shape` carved from one allocation, tensor j starting at
    j * (size + skew) bytes (skew=None: independent allocations)."""
    if skew is None:
        return [torch.empty(shape, dtype=dt, device="cuda") for _ in range(n)]
    eb = torch.empty((), dtype=dt).element_size()
    size = eb
    for e in shape:
        size *= e
    step = size + skew
    big = torch.empty(n * step, dtype=torch.uint8, device="cuda")
    return [big[j * step:j * step + size].view(dt).view(shape) for j in range(n)]


def conv_row(mesh_shape, shape, eb, a, b, peak, tag="", skew=None):
    mesh = Mesh.local(mesh_shape)
    meta = TensorMeta(shape, eb)
    mr = len(mesh_shape)
    s, t = ShardingSpec.parse(a, mr), ShardingSpec.parse(b, mr)
    path = find_transform_path(s, t, mesh.geo, meta)
    dt = {1: torch.uint8, 2: torch.int16, 4: torch.int32, 8: torch.int64}[eb]
    ins = carve(mesh.num_devices, s.local_shape(meta, mesh.geo), dt, skew)
    outs = carve(mesh.num_devices, t.local_shape(meta, mesh.geo), dt, skew)
    tr = mesh.exchange_traffic(s, t, meta)
    nbytes = tr["hbm_read"] + tr["hbm_write"]
    conv = mesh.prepare(path, meta, fuse=True)
    ms = graph_ms(lambda st: conv(ins, outs, stream=st))
    row = {"case": f"{mesh_shape} {list(shape)} e{eb} {a}->{b}{tag}",
           "engine": mesh.exchange_engine(s, t, meta), "alg_bytes": nbytes,
           "us": round(ms * 1e3, 2), "gbs": round(nbytes / ms / 1e6, 1),
           "frac": round(nbytes / ms / 1e6 / peak, 3)}
    conv.close()
    del ins, outs, mesh
    torch.cuda.empty_cache()
    return row


def main():
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] \
        if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
    eng = os.environ.get("APL_COPY_ENGINE", "auto")
    quick = "--quick" in sys.argv
    tag = os.environ.get("PROBE_TAG", "")
    small = "--small" in sys.argv  # launch-bound regime: the block / MLP plans' conversions
    if small:
        for kib in (256, 1024, 4096, 16384):
            n = kib << 9
            x = torch.empty(n, dtype=torch.int16, device="cuda")
            y = torch.empty_like(x)
            ms = graph_ms(lambda st: y.copy_(x))
            print(json.dumps({"case": f"torch copy_ {kib} KiB", "us": round(ms * 1e3, 2)}),
                  flush=True)
            rows = (kib << 10) // (2 * 1024)
            for a, t in (("S0R", "RR"), ("S0R", "RS0"), ("S0R", "S0R")):
                r = conv_row([8], (rows, 1024), 2, a, t, peak)
                print(json.dumps(r), flush=True)
        return
    for mib in ((128, 1024) if quick else (32, 64, 128, 256, 512, 1024)):
        n = mib << 19  # bf16 elements
        x = torch.empty(n, dtype=torch.int16, device="cuda")
        y = torch.empty_like(x)
        ms = graph_ms(lambda st: y.copy_(x))
        if not quick:
          print(json.dumps({"case": f"torch copy_ {mib} MiB", "engine": eng, "us": round(ms * 1e3, 2),
                            "gbs": round(4 * n / ms / 1e6, 1),
                            "frac": round(4 * n / ms / 1e6 / peak, 3)}), flush=True)
        del x, y
        rows = (mib << 20) // (2 * 8192)
        for tgt in ("S0R", "RS0"):
            r = conv_row([8], (rows, 8192), 2, "S0R", tgt, peak)
            r["engine_env"] = eng + tag
            print(json.dumps(r), flush=True)
    for mesh_shape, shape, a, b in ((([2, 2, 2], (8192, 8192), "S012R", "RS012"),
                                      ([2, 4], (8192, 8192), "S01R", "S0S1")) if quick else (
        ([2, 4], (8192, 8192), "S01R", "S1S0"),
        ([2, 4], (8192, 8192), "S0S1", "RS01"),
        ([2, 4], (8192, 8192), "S01R", "S0S1"),
        ([2, 4], (8192, 8192), "RR", "S01R"),
        ([2, 2, 2], (8192, 8192), "S012R", "RS012"),
        ([2, 2, 2], (512, 512, 256), "S0S1R", "RS1S0"),
    )):
        r = conv_row(mesh_shape, shape, 2, a, b, peak)
        r["engine_env"] = eng + tag
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
