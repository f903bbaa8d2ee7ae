"""Per-parameter gradient error of the gpt_block training step under every
reference plan vs fp32 torch autograd (the numbers behind
tests/test_gpu_block.py::test_block_plans_backward), plus forward+backward
step time on one B200 (simulated mesh, one CUDA graph per step).

    python tools/block_grad_check.py
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import torch  # noqa: E402

from paper_2302_02599_b200.executor import PlanExecutor  # noqa: E402
from paper_2302_02599_b200.runtime import Mesh  # noqa: E402
from test_gpu_block import BLOCK_PLANS, PARAMS, PLANS, _case, _reference_grads, _unshard  # noqa: E402


def main():
    for name in BLOCK_PLANS:
        tag = name.split("_mesh")[0].removeprefix("gpt_block_")
        graph, feeds, _ = _case(tag)
        gy, ref = _reference_grads(tag)
        plan = json.loads((PLANS / name).read_text())
        ex = PlanExecutor(Mesh.local(plan["mesh"]["shape"]), graph, plan)
        shards = {k: ex.shard(k, v) for k, v in feeds.items()}
        ex.forward(shards, train=True)
        grads = ex.backward(gy)
        torch.cuda.synchronize()
        errs_grads = {k: _unshard(ex, k, grads[k]).float() for k in PARAMS}
        # timing: the whole training step (forward + backward) as one CUDA graph
        replay, _, _ = ex.capture(shards, grad_out=gy)
        for _ in range(3):
            replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            replay()
        b.record()
        torch.cuda.synchronize()
        errs = {}
        for k in PARAMS:
            g = errs_grads[k]
            r = ref[k]
            errs[k] = (round(((g - r).abs().max() / r.abs().max()).item(), 4),
                       round(((g - r).abs().mean() / r.abs().mean()).item(), 4))
        print(json.dumps({"plan": name.removesuffix(".json"),
                          "train_step_ms_graph": round(a.elapsed_time(b) / 10, 3),
                          "grad_err_max_mean": errs}), flush=True)


if __name__ == "__main__":
    main()
