"""Reference plans (oracle/_ref: the reference's own planner, planner.cpp:91-212)
for a small graph exercising the general transpose and a softmax over a
non-last axis (graph_ir.cpp:270-290; softmax strategies keep the axis
replicated, intraop.cpp:368-384):

    x [B, S, H] -> layernorm(g, b) -> transpose perm [1, 0, 2] -> softmax
    axis 1 -> transpose perm [2, 0, 1] -> output

Writes tests/golden/plans/permute_graph.json and permute_mesh{4,2x2}_unlimited.json.
Run in the build container: make -C oracle && python tests/golden/make_permute_plans.py
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
sys.path.insert(0, str(HERE.parent.parent))

from make_plans import plan  # noqa: E402


def permute_graph(b=8, s=64, h=128, eb=2):
    def node(id_, kind, inputs, shape=None, grad=False, attrs=None):
        n = {"id": id_, "kind": kind, "inputs": [[i, 0] for i in inputs], "outputs": []}
        if shape is not None:
            n["outputs"] = [{"shape": list(shape), "dtype_bytes": eb, "requires_grad": grad}]
        if attrs:
            n["attrs"] = attrs
        return n

    return {"version": 1, "placeholders": ["x"], "output": "out", "nodes": [
        node("x", "placeholder", [], (b, s, h)),
        node("g", "parameter", [], (h,), True),
        node("bb", "parameter", [], (h,), True),
        node("ln", "layernorm", ["x", "g", "bb"]),
        node("t1", "transpose", ["ln"], attrs={"perm": [1, 0, 2]}),
        node("sm", "softmax", ["t1"], attrs={"axis": 1}),
        node("t2", "transpose", ["sm"], attrs={"perm": [2, 0, 1]}),
        node("out", "output", ["t2"])]}


def main():
    out = HERE / "plans"
    g = permute_graph()
    (out / "permute_graph.json").write_text(json.dumps(g, indent=1) + "\n")
    for mesh, tag in (([4], "4"), ([2, 2], "2x2")):
        doc = plan(g, mesh, 1 << 40)
        (out / f"permute_mesh{tag}_unlimited.json").write_text(json.dumps(doc, indent=1) + "\n")
        print(tag, {k: v["strategy"] for k, v in doc["nodes"].items()})


if __name__ == "__main__":
    main()
