"""Transformer-block forward timing on one B200: the reference's gpt_block
graph at GPT-2-medium width (tests/golden/plans/gpt_block_b*_graph.json)
executed from the reference planner's plans on a simulated mesh (every mesh
device a set of buffers on this GPU, so the GPU does all devices' work), as
one CUDA graph per forward. The 1-device plan (everything replicated, no
communication) is the dense baseline: the gap to it is what the plan's
conversions and the extra replicated work cost.

    python tools/block_bench.py [--quick] [--fuse-gather]   # weight all-gathers fused into GEMMs
    python tools/block_bench.py --once gpt_block_b8s1024_mesh8_unlimited   # ncu target
    python tools/block_bench.py --once-train gpt_block_b8s1024_mesh8_unlimited

FLOPs per forward: QKV + proj 4 x 2BSH^2, scores + ctx 2 x 2BS^2H, MLP
2 x 2BSHF (the whole block, all devices together).
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import torch  # noqa: E402

from paper_2302_02599_b200.executor import PlanExecutor  # noqa: E402
from paper_2302_02599_b200.runtime import Mesh, launch_count  # noqa: E402
from test_gpu_block import _operands  # noqa: E402

PLANS = ROOT / "tests" / "golden" / "plans"


def one_device_plan(graph):
    """Every node replicated on a 1-device mesh (the catalog's `replicated`
    matmuls, local non-GEMM strategies): the dense baseline, no conversions."""
    from paper_2302_02599_b200.executor import infer_shapes

    sh = infer_shapes(graph)
    nodes = {}
    prefix = {"reshape": "reshape", "transpose": "perm", "softmax": "softmax",
              "layernorm": "layernorm"}
    for n in graph["nodes"]:
        k = n["kind"]
        if k in ("matmul", "batched-matmul"):
            name = "replicated"
        elif k in prefix:
            name = f"{prefix[k]}:{'R' * len(sh[n['inputs'][0][0]][0])}"
        else:
            name = "local"
        nodes[n["id"]] = {"strategy": name, "spec": "R" * len(sh[n["id"]][0]),
                          "partial_sum": False}
    return {"version": 1, "nodes": nodes, "inserted_comm_nodes": [], "mesh": {"shape": [1]}}


def flops(graph):
    s = {n["id"]: n["outputs"][0]["shape"] for n in graph["nodes"] if n["outputs"]}
    b, sq = s["tok"]
    h = s["wte"][1]
    f = s["w1"][1]
    return 4 * 2.0 * b * sq * h * h + 2 * 2.0 * b * sq * sq * h + 2 * 2.0 * b * sq * h * f


def time_forward(ex, feeds, iters):
    shards = {k: ex.shard(k, v) for k, v in feeds.items()}
    replay, outs, _ = ex.capture(shards)
    torch.cuda.synchronize()
    for _ in range(3):
        replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        replay()
    b.record()
    torch.cuda.synchronize()
    before = launch_count()
    ex.forward(shards)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters, launch_count() - before


def once(stem, train=False):
    """Two eager forwards (train: forward + backward steps) of one plan, for
    an ncu launch list."""
    tag = stem.split("_mesh")[0]
    graph = json.loads((PLANS / f"{tag}_graph.json").read_text())
    plan = json.loads((PLANS / f"{stem}.json").read_text())
    feeds = _operands(graph)
    ex = PlanExecutor(Mesh.local(plan["mesh"]["shape"]), graph, plan)
    shards = {k: ex.shard(k, v) for k, v in feeds.items()}
    gy = torch.randn(feeds["tok"].shape + (feeds["wte"].shape[1],), device="cuda").bfloat16()
    for _ in range(2):
        ex.forward(shards, train=train)
        if train:
            ex.backward(gy)
    torch.cuda.synchronize()


def main():
    if "--once" in sys.argv:
        return once(sys.argv[sys.argv.index("--once") + 1])
    if "--once-train" in sys.argv:
        return once(sys.argv[sys.argv.index("--once-train") + 1], train=True)
    quick = "--quick" in sys.argv
    iters = 5 if quick else 20
    rows = []
    for tag in ("b8s1024", "b4s1024", "b1s4096"):
        graph = json.loads((PLANS / f"gpt_block_{tag}_graph.json").read_text())
        feeds = _operands(graph)
        fl = flops(graph)
        cases = [("1 device (dense)", one_device_plan(graph))]
        for p in sorted(PLANS.glob(f"gpt_block_{tag}_mesh*.json")):
            cases.append((p.stem.split("_mesh")[1], json.loads(p.read_text())))
        for name, plan in cases[:2] if quick else cases:
            shape = plan["mesh"]["shape"]
            mesh = Mesh.local(shape)
            ndev = 1
            for x in shape:
                ndev *= x
            for fuse in ((True,) if ndev == 1 else (True, False)):
                ex = PlanExecutor(mesh, graph, plan, fuse=fuse,
                                  fuse_gather=True if "--fuse-gather" in sys.argv else None)
                ms, launches = time_forward(ex, feeds, iters)
                row = {"graph": tag, "plan": name, "devices": ndev, "fuse": fuse,
                       "ms_per_forward": round(ms, 4), "kernel_launches": launches,
                       # one block's FLOPs per forward (all simulated devices
                       # together compute exactly one block, plus whatever
                       # the plan replicates)
                       "block_tflops": round(fl / (ms * 1e-3) / 1e12, 1)}
                rows.append(row)
                print(json.dumps(row), flush=True)
    return rows


if __name__ == "__main__":
    main()
