"""Regenerate tests/golden/*.json from the REFERENCE library (oracle/_ref).

Run in the build container (needs /root/reference to build oracle/_ref):
    make -C oracle && python tests/golden/make_golden.py

paths.json.gz holds, per case (mesh, tensor shape, dtype bytes), the full
enumeration of valid specs (reference tests/helpers.hpp:245-276) and, for
every ordered pair, the reference path (find_transform_path +
conversion_cost, proj/src/layout.cpp:253-329) with its BFS optimum
(helpers.hpp:344-363). one_step.json holds reference one-step sets
(layout.cpp:162-221); costs.json reference collective_cost values
(cluster.cpp:374-400). The GPU box has no /root/reference, so tests there
check against these committed files.
"""
from __future__ import annotations

import gzip
import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

from oracle import ref  # noqa: E402

# (name, mesh, shape, dtype_bytes, all_pairs)
CASES = [
    ("mesh24_8x8", [2, 4], [8, 8], 4, True),          # test_layout.cpp:148-165, acceptance crit. 1
    ("mesh4_1024sq", [4], [1024, 1024], 4, True),      # test_layout.cpp:198-212
    ("mesh8_rank2", [8], [64, 8192], 2, True),         # config 2
    ("mesh22_1024sq", [2, 2], [1024, 1024], 4, True),  # config 1
    ("mesh24_8192sq_bf16", [2, 4], [8192, 8192], 2, True),  # config 3
    ("mesh222_rank2", [2, 2, 2], [8192, 8192], 2, True),    # config 4 (rank 2)
    ("mesh222_rank2_small", [2, 2, 2], [8, 8], 4, True),
    ("mesh222_rank3_444", [2, 2, 2], [4, 4, 4], 4, True),   # SURVEY Appendix A replay case
    ("mesh222_rank3_small", [2, 2, 2], [8, 4, 2], 4, True),  # test_layout.cpp:264-280
    ("mesh222_rank3", [2, 2, 2], [512, 512, 256], 2, True),  # config 4 (rank 3)
    ("mesh42_1024sq", [4, 2], [1024, 1024], 4, True),
    ("mesh23_12x18", [2, 3], [12, 18], 4, True),        # non-power-of-two extents
]


def main() -> None:
    assert ref.available(), "build oracle/_ref first: make -C oracle"
    cases = []
    for name, mesh, shape, eb, _ in CASES:
        specs = ref.all_valid_specs(mesh, shape, eb)
        pairs = []
        for s in specs:
            for t in specs:
                rc, steps, cost = ref.find_path(mesh, shape, eb, s, t)
                assert rc == 0, (name, s, t, steps)
                bfs = ref.bfs_min_steps(mesh, shape, eb, s, t)
                pairs.append([s, t, [list(x) for x in steps], repr(cost), bfs])
        cases.append({"name": name, "mesh": mesh, "shape": shape, "dtype_bytes": eb,
                      "specs": specs, "pairs": pairs})
        print(f"{name}: {len(specs)} specs, {len(pairs)} pairs", file=sys.stderr)
    with gzip.open(HERE / "paths.json.gz", "wt") as f:
        json.dump({"cases": cases}, f, separators=(",", ":"))

    one = []
    for mesh, shape, eb, spec in [([2, 4], [8, 8], 4, "S0R"), ([2, 4], [8, 8], 4, "RR"),
                                  ([2, 4], [3, 8], 4, "RR"), ([2, 2, 2], [8, 4, 2], 4, "S0S1R"),
                                  ([2, 4], [8192, 8192], 2, "S01R"), ([8], [64, 8192], 2, "S0R")]:
        rc, out = ref.one_step(mesh, shape, eb, spec)
        assert rc == 0
        one.append({"mesh": mesh, "shape": shape, "dtype_bytes": eb, "spec": spec,
                    "neighbours": [list(x) for x in out]})
    (HERE / "one_step.json").write_text(json.dumps(one, indent=0))

    costs = []
    for mesh, axes, kind, nbytes in [([4], [0], 0, 1048576), ([4], [0], 1, 1 << 20),
                                     ([4], [0], 2, 1 << 20), ([2, 4], [0, 1], 1, 12345.0),
                                     ([2, 4], [1], 3, 16 << 20), ([2, 4], [0], 4, 99.0),
                                     ([1, 4], [0], 0, 1024.0), ([2, 2, 2], [0, 2], 3, 777.0)]:
        rc, v = ref.collective_cost(mesh, axes, kind, nbytes)
        assert rc == 0
        costs.append({"mesh": mesh, "axes": axes, "kind": kind, "bytes": nbytes,
                      "cost": repr(v)})
    (HERE / "costs.json").write_text(json.dumps(costs, indent=0))


if __name__ == "__main__":
    main()
