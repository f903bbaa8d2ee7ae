"""Run one conversion a few times eagerly (an ncu target).

    python tools/ncu_case.py 2,2,2 8192,8192 2 S012R RS012 [reps]
"""
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
    eb = int(sys.argv[3])
    a, b = sys.argv[4], sys.argv[5]
    reps = int(sys.argv[6]) if len(sys.argv) > 6 else 3
    mesh = Mesh.local(ms)
    meta = TensorMeta(shape, eb)
    s, t = ShardingSpec.parse(a, len(ms)), ShardingSpec.parse(b, len(ms))
    path = find_transform_path(s, t, mesh.geo, meta)
    dt = {1: torch.uint8, 2: torch.int16, 4: torch.int32, 8: torch.int64}[eb]
    ins = [torch.empty(s.local_shape(meta, mesh.geo), dtype=dt, device="cuda")
           for _ in range(mesh.num_devices)]
    outs = [torch.empty(t.local_shape(meta, mesh.geo), dtype=dt, device="cuda")
            for _ in range(mesh.num_devices)]
    conv = mesh.prepare(path, meta, fuse=True)
    for _ in range(reps):
        conv(ins, outs)
    torch.cuda.synchronize()
    print("engine", mesh.exchange_engine(s, t, meta), mesh.exchange_traffic(s, t, meta))


if __name__ == "__main__":
    main()
