"""Time one conversion (collapsed, prepared) under the current APL_* knobs:
prints {"pair", "engine", "us", "frac", "env"}. The knob sweep for a slow
class runs this once per setting (each knob is read once per process).

    APL_COPY_VARIANT=0 python tools/pair_probe.py 2,4 8192,8192 S01R RS1
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


def main():
    ms = [int(x) for x in sys.argv[1].split(",")]
    shape = tuple(int(x) for x in sys.argv[2].split(","))
    a, b = sys.argv[3], sys.argv[4]
    iters = int(sys.argv[5]) if len(sys.argv) > 5 else 20
    mesh = Mesh.local(ms)
    meta = TensorMeta(shape, 2)
    s, t = ShardingSpec.parse(a, len(ms)), ShardingSpec.parse(b, len(ms))
    conv = mesh.prepare(find_transform_path(s, t, mesh.geo, meta), meta, fuse=True)
    ins = [torch.empty(s.local_shape(meta, mesh.geo), dtype=torch.int16, device="cuda")
           .random_(-3000, 3000) for _ in range(mesh.num_local)]
    outs = [torch.empty(t.local_shape(meta, mesh.geo), dtype=torch.int16, device="cuda")
            for _ in range(mesh.num_local)]
    tr = mesh.exchange_traffic(s, t, meta)
    nbytes = tr["hbm_read"] + tr["hbm_write"]
    st = torch.cuda.current_stream()
    for _ in range(3):
        conv(ins, outs, stream=st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(iters):
        conv(ins, outs, stream=st)
    e1.record(st)
    torch.cuda.synchronize()
    ms_ = e0.elapsed_time(e1) / iters
    env = {k: v for k, v in os.environ.items() if k.startswith("APL_")}
    print(json.dumps({"pair": f"{a}->{b}", "mesh": ms, "tensor": list(shape),
                      "engine": mesh.exchange_engine(s, t, meta), "us": round(ms_ * 1e3, 2),
                      "frac": round(nbytes / (ms_ * 1e-3) / 1e9 / 6457.1, 4), "env": env}))


if __name__ == "__main__":
    main()
