"""BASELINE config 5 timing on one B200 (simulated 8-device mesh): the
GPT-2-medium MLP forward executed from the reference planner's plans and the
pinned Megatron plan. Reports ms per forward, the GEMM / conversion split
and TFLOP/s of the whole step (2 GEMMs x 2*16384*1024*4096 FLOPs, all 8
simulated devices together = one GPU doing 8 devices' work).

    python tools/mlp_bench.py [--quick]
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2302_02599_b200.executor import PlanExecutor, megatron_mlp_plan  # noqa: E402
from paper_2302_02599_b200.runtime import Mesh  # noqa: E402

PLANS = ROOT / "tests" / "golden" / "plans"
GRAPH = json.loads((PLANS / "gpt2_mlp_graph.json").read_text())
FLOPS = 2 * 2.0 * 16384 * 1024 * 4096
# training step: forward (2 GEMMs) + backward (fc2 dA and dB, fc1 dB; the
# input x needs no gradient) = 5 GEMMs of 2*16384*1024*4096
TRAIN_FLOPS = 5 * 2.0 * 16384 * 1024 * 4096


def main():
    quick = "--quick" in sys.argv
    torch.manual_seed(0)
    feeds = {"x": torch.randn(16384, 1024, device="cuda").bfloat16(),
             "w1": (torch.randn(1024, 4096, device="cuda") / 32).bfloat16(),
             "w2": (torch.randn(4096, 1024, device="cuda") / 64).bfloat16()}
    plans = [("megatron [8]", megatron_mlp_plan(), [8])]
    for p in sorted(PLANS.glob("gpt2_mlp_mesh*unlimited.json")):
        doc = json.loads(p.read_text())
        plans.append((f"reference {p.stem}", doc, doc["mesh"]["shape"]))
    iters = 3 if quick else 20
    for name, plan, shape in plans[:2] if quick else plans:
        mesh = Mesh.local(shape)
        for fuse in (True, False):
            ex = PlanExecutor(mesh, GRAPH, plan, fuse=fuse)
            shards = {k: ex.shard(k, v) for k, v in feeds.items()}
            for _ in range(3):
                ex.forward(shards)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(iters):
                ex.forward(shards)
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / iters
            gy = torch.randn(16384, 1024, device="cuda").bfloat16()

            def step():
                ex.forward(shards, train=True)
                ex.backward(gy)

            for _ in range(3):
                step()
            torch.cuda.synchronize()
            a.record()
            for _ in range(iters):
                step()
            b.record()
            torch.cuda.synchronize()
            tms = a.elapsed_time(b) / iters
            # the same steps captured in CUDA graphs (device time, no host
            # launch overhead): every kernel of the executor is stream-ordered
            # on the capture stream and everything is compiled by the warm-up
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            graphs = {}
            with torch.cuda.stream(side):
                ex.forward(shards, stream=side)
                ex.forward(shards, stream=side, train=True)
                ex.backward(gy, stream=side)
                side.synchronize()
                gf, gt = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
                with torch.cuda.graph(gf, stream=side):
                    ex.forward(shards, stream=side)
                with torch.cuda.graph(gt, stream=side):
                    ex.forward(shards, stream=side, train=True)
                    ex.backward(gy, stream=side)
                graphs = {"fwd": gf, "train": gt}
            torch.cuda.current_stream().wait_stream(side)
            gms = {}
            for k, g in graphs.items():
                g.replay()
                torch.cuda.synchronize()
                a.record()
                for _ in range(iters):
                    g.replay()
                b.record()
                torch.cuda.synchronize()
                gms[k] = a.elapsed_time(b) / iters
            print(json.dumps({"plan": name, "fuse": fuse, "ms_per_forward": round(ms, 4),
                              "tflops": round(FLOPS / ms / 1e9, 1),
                              "ms_per_train_step": round(tms, 4),
                              "train_tflops": round(TRAIN_FLOPS / tms / 1e9, 1),
                              "graph_ms_per_forward": round(gms["fwd"], 4),
                              "graph_tflops": round(FLOPS / gms["fwd"] / 1e9, 1),
                              "graph_ms_per_train_step": round(gms["train"], 4),
                              "graph_train_tflops": round(TRAIN_FLOPS / gms["train"] / 1e9, 1),
                              "strategies": {k: v.name for k, v in ex.strategy.items()}}),
                  flush=True)


if __name__ == "__main__":
    main()
