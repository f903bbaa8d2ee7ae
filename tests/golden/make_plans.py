"""Regenerate tests/golden/{strategies,plans}/ from the REFERENCE planner
(oracle/_ref). Run in the build container:

    make -C oracle && python tests/golden/make_plans.py

strategies.json : the reference catalog (generate_strategies,
                  proj/src/intraop.cpp:141-234, 497-555, 719-767) for the
                  GPT-2-medium MLP matmuls and a rank-3 batched case.
plans/*.json    : version-1 plan documents (plan_to_json, planner.cpp:455-600)
                  of the reference's full sweep (planner.cpp:91-212) for
                  BASELINE config 5 on an 8-GPU uniform NVSwitch mesh
                  (alpha 3 us, 900 GB/s, 1.65 PFLOP/s per device), with the
                  graph document they were planned from;
                  gpt_block_*: the same for the reference's transformer-block
                  graph (proj/tests/fixtures/gpt_block.json) -- the fixture
                  itself ("fixture", fp32 [4,16,64]) and a GPT-2-medium-width
                  bf16 instances ("b8s1024": batch 8, seq 1024, hidden 1024,
                  vocab 50304, MLP 4096; "b4s1024", "b1s4096": smaller
                  batches, which make the planner shard sequence / hidden
                  dims instead), same node ids and kinds.
"""
from __future__ import annotations

import ctypes as C
import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

from oracle import ref  # noqa: E402

ALPHA, BETA_INV, FLOPS = 3e-6, 1.0 / 900e9, 1.65e15


def mlp_graph(tokens=16384, d=1024, hidden=4096, dtype_bytes=2):
    def node(id_, kind, inputs, shape=None, grad=False):
        n = {"id": id_, "kind": kind, "inputs": [[i, 0] for i in inputs], "outputs": []}
        if shape is not None:
            n["outputs"] = [{"shape": list(shape), "dtype_bytes": dtype_bytes,
                             "requires_grad": grad}]
        return n

    return {"version": 1, "placeholders": ["x"], "output": "out", "nodes": [
        node("x", "placeholder", [], (tokens, d)),
        node("w1", "parameter", [], (d, hidden), True),
        node("w2", "parameter", [], (hidden, d), True),
        node("fc1", "matmul", ["x", "w1"]),
        node("gelu", "elementwise-unary", ["fc1"]),
        node("fc2", "matmul", ["gelu", "w2"]),
        node("out", "output", ["fc2"]),
    ]}


def bmm_graph():
    def node(id_, kind, inputs, shape=None, grad=False):
        n = {"id": id_, "kind": kind, "inputs": [[i, 0] for i in inputs], "outputs": []}
        if shape is not None:
            n["outputs"] = [{"shape": list(shape), "dtype_bytes": 2, "requires_grad": grad}]
        return n

    return {"version": 1, "placeholders": ["a", "b"], "output": "out", "nodes": [
        node("a", "placeholder", [], (16, 64, 32)), node("b", "placeholder", [], (16, 32, 48)),
        node("bmm", "batched-matmul", ["a", "b"]), node("out", "output", ["bmm"])]}


def block_graph(b=8, s=1024, h=1024, v=50304, f=4096, eb=2):
    """The reference's gpt_block graph (proj/tests/fixtures/gpt_block.json:
    same ids, kinds, edges and attrs) at other sizes; ids int64, mask u8."""
    def node(id_, kind, inputs, shape=None, grad=False, dtype=eb, attrs=None):
        n = {"id": id_, "kind": kind, "inputs": [[i, 0] for i in inputs], "outputs": []}
        if shape is not None:
            n["outputs"] = [{"shape": list(shape), "dtype_bytes": dtype, "requires_grad": grad}]
        if attrs:
            n["attrs"] = attrs
        return n

    bsh = {"target_shape": [b, s, h]}
    flat = {"target_shape": [b * s, h]}
    nodes = [node("tok", "placeholder", [], (b, s), dtype=8),
             node("mask", "placeholder", [], (b, s, s), dtype=1),
             node("wte", "parameter", [], (v, h), True)]
    for p, shape in (("g1", (h,)), ("b1", (h,)), ("wq", (h, h)), ("wk", (h, h)), ("wv", (h, h)),
                     ("wo", (h, h)), ("g2", (h,)), ("b2", (h,)), ("w1", (h, f)), ("w2", (f, h))):
        nodes.append(node(p, "parameter", [], shape, True))
    nodes += [
        node("emb", "embedding-lookup", ["tok", "wte"]),
        node("ln1", "layernorm", ["emb", "g1", "b1"]),
        node("r1", "reshape", ["ln1"], attrs=flat),
        node("q2", "matmul", ["r1", "wq"]), node("k2", "matmul", ["r1", "wk"]),
        node("v2", "matmul", ["r1", "wv"]),
        node("qr", "reshape", ["q2"], attrs=bsh), node("kr", "reshape", ["k2"], attrs=bsh),
        node("vr", "reshape", ["v2"], attrs=bsh),
        node("kt", "transpose", ["kr"], attrs={"perm": [0, 2, 1]}),
        node("scores", "batched-matmul", ["qr", "kt"]),
        node("scaled", "elementwise-unary", ["scores"]),
        node("mask2", "elementwise-unary", ["mask"]),
        node("att_in", "elementwise-binary", ["scaled", "mask2"]),
        node("att", "softmax", ["att_in"], attrs={"axis": -1}),
        node("ctx", "batched-matmul", ["att", "vr"]),
        node("r2", "reshape", ["ctx"], attrs=flat), node("po", "matmul", ["r2", "wo"]),
        node("pr", "reshape", ["po"], attrs=bsh),
        node("res1", "elementwise-binary", ["pr", "emb"]),
        node("ln2", "layernorm", ["res1", "g2", "b2"]),
        node("r3", "reshape", ["ln2"], attrs=flat), node("h1", "matmul", ["r3", "w1"]),
        node("act", "elementwise-unary", ["h1"]), node("h2", "matmul", ["act", "w2"]),
        node("mr", "reshape", ["h2"], attrs=bsh),
        node("res2", "elementwise-binary", ["mr", "res1"]),
        node("out", "output", ["res2"])]
    return {"version": 1, "placeholders": ["tok", "mask"], "output": "out", "nodes": nodes}


def node_strategies(graph, node_id, mesh):
    lib = ref.lib()
    lib.ref_node_strategies.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(C.c_int64), C.c_int,
                                        C.c_double, C.c_char_p, C.c_size_t]
    buf = C.create_string_buffer(1 << 20)
    rc = lib.ref_node_strategies(json.dumps(graph).encode(), node_id.encode(),
                                 (C.c_int64 * len(mesh))(*mesh), len(mesh), FLOPS, buf, len(buf))
    assert rc == 0, buf.value
    rows = []
    for line in buf.value.decode().splitlines():
        name, a, b, c, partial, red, comp, comm, mem = line.split("|")
        rows.append({"name": name, "a": a, "b": b, "c": c, "partial_sum": partial == "1",
                     "reduce_axes": [int(x) for x in red.split(",") if x],
                     "compute_time_s": comp, "comm_time_s": comm, "memory_bytes": int(mem)})
    return rows


def plan(graph, mesh, budget):
    lib = ref.lib()
    lib.ref_plan.argtypes = [C.c_char_p, C.POINTER(C.c_int64), C.c_int, C.c_double, C.c_double,
                             C.c_double, C.c_int64, C.c_char_p, C.c_size_t]
    buf = C.create_string_buffer(1 << 24)
    rc = lib.ref_plan(json.dumps(graph).encode(), (C.c_int64 * len(mesh))(*mesh), len(mesh),
                      ALPHA, BETA_INV, FLOPS, budget, buf, len(buf))
    assert rc == 0, buf.value[:500]
    return json.loads(buf.value.decode())


def main():
    assert ref.available(), "build oracle/_ref first: make -C oracle"
    g = mlp_graph()
    strategies = []
    for mesh in ([8], [2, 4], [2, 2, 2]):
        for nid in ("fc1", "fc2"):
            strategies.append({"graph": "gpt2_mlp", "node": nid, "mesh": mesh,
                               "flops": FLOPS, "strategies": node_strategies(g, nid, mesh)})
    strategies.append({"graph": "bmm", "node": "bmm", "mesh": [2, 2], "flops": FLOPS,
                       "strategies": node_strategies(bmm_graph(), "bmm", [2, 2])})
    (HERE / "strategies.json").write_text(json.dumps({"graphs": {"gpt2_mlp": g, "bmm": bmm_graph()},
                                                      "cases": strategies}, indent=0))
    out = HERE / "plans"
    out.mkdir(exist_ok=True)
    (out / "gpt2_mlp_graph.json").write_text(json.dumps(g, indent=1))
    for mesh in ([8], [2, 4], [2, 2, 2]):
        for budget_mib in (0, 88, 96, 192):  # 88: Rotor checkpoints fc1/gelu
            budget = (budget_mib << 20) if budget_mib else (1 << 40)
            name = f"gpt2_mlp_mesh{'x'.join(map(str, mesh))}_{budget_mib or 'unlimited'}"
            try:
                doc = plan(g, mesh, budget)
            except AssertionError as e:
                print(f"{name}: infeasible ({e})", file=sys.stderr)
                continue
            (out / f"{name}.json").write_text(json.dumps(doc, indent=1))
            sel = {k: v["strategy"] for k, v in doc["nodes"].items()}
            comm = [(c["node"], c["collective"], c["axes"]) for c in doc["inserted_comm_nodes"]]
            print(name, sel, comm, file=sys.stderr)
    fixture = json.loads(Path("/root/reference/proj/tests/fixtures/gpt_block.json").read_text())
    blocks = {"fixture": (fixture, ([2, 2], [4], [2, 4], [8]), (0,)),
              "b8s1024": (block_graph(), ([8], [2, 4], [2, 2, 2]), (0,)),
              # 100 MiB on [8]: the attention stage is checkpointed (store_boundary)
              "b4s1024": (block_graph(b=4), ([8], [2, 4], [2, 2, 2]), (0, 100)),
              "b1s4096": (block_graph(b=1, s=4096), ([8], [2, 4], [2, 2, 2]), (0,))}
    for tag, (g, meshes, budgets) in blocks.items():
        (out / f"gpt_block_{tag}_graph.json").write_text(json.dumps(g, indent=1))
        for mesh in meshes:
            for budget_mib in budgets:
                budget = (budget_mib << 20) if budget_mib else (1 << 40)
                name = f"gpt_block_{tag}_mesh{'x'.join(map(str, mesh))}_{budget_mib or 'unlimited'}"
                try:
                    doc = plan(g, mesh, budget)
                except AssertionError as e:
                    print(f"{name}: infeasible ({e})", file=sys.stderr)
                    continue
                (out / f"{name}.json").write_text(json.dumps(doc, indent=1))
                print(name, len(doc["inserted_comm_nodes"]), "comm nodes", file=sys.stderr)


if __name__ == "__main__":
    main()
