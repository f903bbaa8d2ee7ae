"""One Megatron-plan forward + training step of the GPT-2-medium MLP on a
simulated [8] mesh (ncu target: python tools/mlp_once.py [plan.json])."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2302_02599_b200.executor import PlanExecutor, megatron_mlp_plan  # noqa: E402
from paper_2302_02599_b200.runtime import Mesh  # noqa: E402

GRAPH = json.loads((ROOT / "tests" / "golden" / "plans" / "gpt2_mlp_graph.json").read_text())


def main():
    plan = json.loads(Path(sys.argv[1]).read_text()) if len(sys.argv) > 1 else megatron_mlp_plan()
    mesh = Mesh.local(plan["mesh"]["shape"] if "mesh" in plan else [8])
    torch.manual_seed(0)
    feeds = {"x": torch.randn(16384, 1024, device="cuda").bfloat16(),
             "w1": (torch.randn(1024, 4096, device="cuda") / 32).bfloat16(),
             "w2": (torch.randn(4096, 1024, device="cuda") / 64).bfloat16()}
    ex = PlanExecutor(mesh, GRAPH, plan)
    shards = {k: ex.shard(k, v) for k, v in feeds.items()}
    gy = torch.randn(16384, 1024, device="cuda").bfloat16()
    for _ in range(2):
        ex.forward(shards)
        ex.forward(shards, train=True)
        ex.backward(gy)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
