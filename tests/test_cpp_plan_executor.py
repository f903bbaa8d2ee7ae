"""The native C++ PlanExecutor (include/autoplan/plan_executor.hpp) runs the
reference planner's GPT-2-medium MLP plans and produces exactly the bytes of
the Python PlanExecutor (same kernels, same order) -- and both match fp32
torch within the config-5 tolerance."""
import json
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
PLANS = ROOT / "tests" / "golden" / "plans"
NLOHMANN = Path("/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty")


def build(tmp_path):
    exe = tmp_path / "plan_executor_test"
    lib = ROOT / "paper_2302_02599_b200"
    cmd = ["g++", "-std=c++20", "-O1", f"-I{ROOT / 'include'}", f"-I{NLOHMANN}",
           "-I/usr/local/cuda/include", str(ROOT / "tests/cpp/plan_executor_test.cpp"),
           f"-L{lib}", "-lapl", "-L/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{lib}",
           "-Wl,-rpath,/usr/local/cuda/lib64", "-o", str(exe)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


@pytest.mark.skipif(not NLOHMANN.exists(), reason="nlohmann/json headers not in this image")
def test_plan_executor_header_compiles(tmp_path):
    build(tmp_path)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["gpt2_mlp_mesh8_unlimited.json", "gpt2_mlp_mesh2x4_96.json",
                                  "gpt2_mlp_mesh2x2x2_unlimited.json"])
def test_native_executor_matches_python_executor(cuda, tmp_path, name):
    import torch

    from paper_2302_02599_b200.executor import PlanExecutor
    from paper_2302_02599_b200.runtime import Mesh

    exe = build(tmp_path)
    torch.manual_seed(2302)
    feeds = {"x": torch.randn(16384, 1024, device="cuda").bfloat16(),
             "w1": (torch.randn(1024, 4096, device="cuda") / 32).bfloat16(),
             "w2": (torch.randn(4096, 1024, device="cuda") / 64).bfloat16()}
    for k, v in feeds.items():
        (tmp_path / f"{k}.bin").write_bytes(v.view(torch.int16).cpu().numpy().tobytes())
    plan = json.loads((PLANS / name).read_text())
    mesh_arg = "x".join(map(str, plan["mesh"]["shape"]))
    r = subprocess.run([str(exe), str(PLANS / "gpt2_mlp_graph.json"), str(PLANS / name), mesh_arg,
                        str(tmp_path)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    native = (tmp_path / "out.bin").read_bytes()
    mesh = Mesh.local(plan["mesh"]["shape"])
    ex = PlanExecutor(mesh, json.loads((PLANS / "gpt2_mlp_graph.json").read_text()), plan)
    out = ex.forward(feeds)[0]
    torch.cuda.synchronize()
    assert out.view(torch.int16).cpu().numpy().tobytes() == native
    ref = torch.nn.functional.gelu(feeds["x"].float() @ feeds["w1"].float()) @ feeds["w2"].float()
    assert ((out.double() - ref.double()).abs().max() / ref.abs().max()).item() <= 2e-2


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["gpt_block_b8s1024_mesh8_unlimited.json",
                                  "gpt_block_b4s1024_mesh2x4_unlimited.json",
                                  "gpt_block_b8s1024_mesh2x2x2_unlimited.json",
                                  "gpt_block_b1s4096_mesh2x2x2_unlimited.json"])
def test_native_executor_runs_block_plans(cuda, tmp_path, name):
    """The transformer block (embedding, layernorm, batched matmul, softmax,
    the fused attention chain and owner-block table reads) from the native
    executor: the same bytes as the Python executor."""
    import sys

    import torch

    sys.path.insert(0, str(ROOT / "tests"))
    from test_gpu_block import _operands

    from paper_2302_02599_b200.executor import PlanExecutor
    from paper_2302_02599_b200.runtime import Mesh

    exe = build(tmp_path)
    tag = name.split("_mesh")[0]
    graph_path = PLANS / f"{tag}_graph.json"
    graph = json.loads(graph_path.read_text())
    feeds = _operands(graph)
    for k, v in feeds.items():
        (tmp_path / f"{k}.bin").write_bytes(v.contiguous().view(torch.uint8).cpu().numpy()
                                            .tobytes())
    plan = json.loads((PLANS / name).read_text())
    mesh_arg = "x".join(map(str, plan["mesh"]["shape"]))
    r = subprocess.run([str(exe), str(graph_path), str(PLANS / name), mesh_arg, str(tmp_path)],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    native = (tmp_path / "out.bin").read_bytes()
    ex = PlanExecutor(Mesh.local(plan["mesh"]["shape"]), graph, plan)
    out = ex.forward(feeds)[0]
    torch.cuda.synchronize()
    assert out.contiguous().view(torch.uint8).cpu().numpy().tobytes() == native


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["gpt2_mlp_mesh8_unlimited.json", "gpt2_mlp_mesh2x2x2_unlimited.json",
                                  "gpt_block_b8s1024_mesh8_unlimited.json",
                                  "gpt_block_b4s1024_mesh2x4_unlimited.json",
                                  "gpt_block_b8s1024_mesh2x2x2_unlimited.json"])
def test_native_executor_backward_matches_python(cuda, tmp_path, name):
    """Training step from the native executor: every parameter gradient
    (fp32, plan layout, all devices) byte-identical to the Python
    PlanExecutor.backward on the same plan and operands -- except the
    embedding table's, accumulated with fp32 atomics (repeated ids), whose
    summation order is not fixed even between two runs of the same executor:
    within 1e-5 of the largest entry."""
    import sys

    import torch

    sys.path.insert(0, str(ROOT / "tests"))
    from test_gpu_block import _operands

    from paper_2302_02599_b200.executor import PlanExecutor
    from paper_2302_02599_b200.runtime import Mesh

    exe = build(tmp_path)
    tag = name.split("_mesh")[0]
    graph_path = PLANS / f"{tag}_graph.json"
    graph = json.loads(graph_path.read_text())
    if tag == "gpt2_mlp":
        torch.manual_seed(2302)
        feeds = {"x": torch.randn(16384, 1024, device="cuda").bfloat16(),
                 "w1": (torch.randn(1024, 4096, device="cuda") / 32).bfloat16(),
                 "w2": (torch.randn(4096, 1024, device="cuda") / 64).bfloat16()}
        out_shape = (16384, 1024)
    else:
        feeds = _operands(graph)
        out_shape = tuple(feeds["tok"].shape) + (feeds["wte"].shape[1],)
    torch.manual_seed(7)
    gy = torch.randn(out_shape, device="cuda").bfloat16()
    for k, v in feeds.items():
        (tmp_path / f"{k}.bin").write_bytes(v.contiguous().view(torch.uint8).cpu().numpy()
                                            .tobytes())
    (tmp_path / "dy.bin").write_bytes(gy.view(torch.uint8).cpu().numpy().tobytes())
    plan = json.loads((PLANS / name).read_text())
    mesh_arg = "x".join(map(str, plan["mesh"]["shape"]))
    r = subprocess.run([str(exe), str(graph_path), str(PLANS / name), mesh_arg, str(tmp_path),
                        "train"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    ex = PlanExecutor(Mesh.local(plan["mesh"]["shape"]), graph, plan)
    ex.forward(feeds, train=True)
    grads = ex.backward(gy)
    torch.cuda.synchronize()
    assert grads
    for k, shards in grads.items():  # every gradient, the embedding table's included
        mine = b"".join(t.contiguous().view(torch.uint8).cpu().numpy().tobytes() for t in shards)
        native = (tmp_path / f"grad_{k}.bin").read_bytes()
        assert native == mine, k


@pytest.mark.gpu
def test_native_training_forward_rejects_fp32_plans(cuda, tmp_path):
    """The native backward computes in bf16: a training forward of the
    reference's fp32 fixture plan (every parameter dtype_bytes 4) is refused
    up front with a PlanError, before any kernel reads an fp32
    buffer as bf16. The operands are written at the graph's own widths."""
    import sys

    import torch

    sys.path.insert(0, str(ROOT / "tests"))
    from test_gpu_block import _operands

    exe = build(tmp_path)
    graph_path = PLANS / "gpt_block_fixture_graph.json"
    graph = json.loads(graph_path.read_text())
    widths = {n["id"]: n["outputs"][0]["dtype_bytes"] for n in graph["nodes"] if n["outputs"]}
    feeds = _operands(graph)
    for k, v in feeds.items():
        if v.is_floating_point() and widths[k] == 4:
            v = v.float()
        assert v.element_size() == widths[k], k
        (tmp_path / f"{k}.bin").write_bytes(v.contiguous().view(torch.uint8).cpu().numpy()
                                            .tobytes())
    out_shape = tuple(feeds["tok"].shape) + (feeds["wte"].shape[1],)
    (tmp_path / "dy.bin").write_bytes(torch.zeros(out_shape, dtype=torch.bfloat16)
                                      .view(torch.uint8).numpy().tobytes())
    name = "gpt_block_fixture_mesh2x2_unlimited.json"
    args = [str(exe), str(graph_path), str(PLANS / name), "2x2", str(tmp_path), "train"]
    r = subprocess.run(args, capture_output=True, text=True, timeout=300)
    assert r.returncode != 0
    assert r.returncode != -11, "segfault instead of a PlanError"
    assert "backward supports bf16 plans only" in r.stdout + r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["permute_mesh4_unlimited.json", "permute_mesh2x2_unlimited.json"])
def test_native_executor_general_transpose_and_softmax_axis(cuda, tmp_path, name):
    """The reference planner's plans for a graph with a general transpose
    (perm [1,0,2], [2,0,1]) and a softmax over axis 1
    (tests/golden/make_permute_plans.py): native forward output and every
    parameter gradient byte-identical to the Python executor."""
    import torch

    from paper_2302_02599_b200.executor import PlanExecutor
    from paper_2302_02599_b200.runtime import Mesh

    exe = build(tmp_path)
    graph_path = PLANS / "permute_graph.json"
    graph = json.loads(graph_path.read_text())
    torch.manual_seed(11)
    feeds = {"x": torch.randn(8, 64, 128, device="cuda").bfloat16(),
             "g": (1 + 0.1 * torch.randn(128, device="cuda")).bfloat16(),
             "bb": (0.1 * torch.randn(128, device="cuda")).bfloat16()}
    gy = torch.randn(128, 64, 8, device="cuda").bfloat16()
    for k, v in feeds.items():
        (tmp_path / f"{k}.bin").write_bytes(v.contiguous().view(torch.uint8).cpu().numpy()
                                            .tobytes())
    (tmp_path / "dy.bin").write_bytes(gy.view(torch.uint8).cpu().numpy().tobytes())
    plan = json.loads((PLANS / name).read_text())
    mesh_arg = "x".join(map(str, plan["mesh"]["shape"]))
    r = subprocess.run([str(exe), str(graph_path), str(PLANS / name), mesh_arg, str(tmp_path),
                        "train"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    ex = PlanExecutor(Mesh.local(plan["mesh"]["shape"]), graph, plan)
    out = ex.forward(feeds, train=True)[0]
    grads = ex.backward(gy)
    torch.cuda.synchronize()
    assert out.contiguous().view(torch.uint8).cpu().numpy().tobytes() == \
        (tmp_path / "out.bin").read_bytes()
    assert set(grads) == {"g", "bb"}
    for k, shards in grads.items():
        mine = b"".join(t.contiguous().view(torch.uint8).cpu().numpy().tobytes() for t in shards)
        assert (tmp_path / f"grad_{k}.bin").read_bytes() == mine, k


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["permute_mesh4_unlimited.json", "permute_mesh2x2_unlimited.json",
                                  "gpt2_mlp_mesh8_unlimited.json"])
def test_native_executor_distributed_over_nccl(cuda, tmp_path, name):
    """The native PlanExecutor as one process per mesh device on the NCCL
    transport (MeshRuntime::Distributed: ncclCommSplit per mesh-axis subset,
    all-gather / all-to-all / grouped send-recv conversions, all-reduce of
    partial sums), ranks sharing one GPU through per-rank NCCL_HOSTID over
    the socket transport: every rank's forward output equals the simulated
    mesh's bytes (no reductions in these forwards) and every gradient shard
    matches within fp32 summation order (5e-5 of the largest entry)."""
    import ctypes as C
    import os

    import numpy as np
    import torch

    from paper_2302_02599_b200 import _capi as A

    exe = build(tmp_path)
    tag = name.split("_mesh")[0]
    graph_path = PLANS / f"{tag}_graph.json"
    plan = json.loads((PLANS / name).read_text())
    mesh_shape = plan["mesh"]["shape"]
    P = int(np.prod(mesh_shape))
    if tag == "gpt2_mlp":
        torch.manual_seed(2302)
        feeds = {"x": torch.randn(16384, 1024, device="cuda").bfloat16(),
                 "w1": (torch.randn(1024, 4096, device="cuda") / 32).bfloat16(),
                 "w2": (torch.randn(4096, 1024, device="cuda") / 64).bfloat16()}
        out_shape = (16384, 1024)
    else:
        torch.manual_seed(11)
        feeds = {"x": torch.randn(8, 64, 128, device="cuda").bfloat16(),
                 "g": (1 + 0.1 * torch.randn(128, device="cuda")).bfloat16(),
                 "bb": (0.1 * torch.randn(128, device="cuda")).bfloat16()}
        out_shape = (128, 64, 8)
    gy = torch.randn(out_shape, device="cuda").bfloat16()
    for k, v in feeds.items():
        (tmp_path / f"{k}.bin").write_bytes(v.contiguous().view(torch.uint8).cpu().numpy()
                                            .tobytes())
    (tmp_path / "dy.bin").write_bytes(gy.view(torch.uint8).cpu().numpy().tobytes())
    mesh_arg = "x".join(map(str, mesh_shape))
    args = [str(exe), str(graph_path), str(PLANS / name), mesh_arg, str(tmp_path), "train"]
    r = subprocess.run(args, capture_output=True, text=True, timeout=600)  # simulated reference
    assert r.returncode == 0, r.stdout + r.stderr
    uid = (C.c_uint8 * 128)()
    assert A.lib().apl_nccl_unique_id(uid) == 0
    (tmp_path / "nccl.id").write_bytes(bytes(uid))
    procs = []
    for rank in range(P):
        env = dict(os.environ, APL_TEST_RANK=str(rank), APL_TEST_IDFILE=str(tmp_path / "nccl.id"),
                   NCCL_HOSTID=f"apl-native-host-{rank}", NCCL_SOCKET_IFNAME="lo",
                   NCCL_IB_DISABLE="1")
        procs.append(subprocess.Popen(args, env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=900) for p in procs]
    assert all(p.returncode == 0 for p in procs), [o[1][-2000:] for o in outs]
    ref_out = (tmp_path / "out.bin").read_bytes()
    for rank in range(P):
        assert (tmp_path / f"out_r{rank}.bin").read_bytes() == ref_out, rank
    grads = [k for k in feeds if k != "x"]  # the parameters
    for gid in grads:
        ref = np.frombuffer((tmp_path / f"grad_{gid}.bin").read_bytes(), dtype=np.float32)
        per = ref.size // P
        scale = float(np.abs(ref).max()) or 1.0
        for rank in range(P):
            mine = np.frombuffer((tmp_path / f"grad_{gid}_r{rank}.bin").read_bytes(),
                                 dtype=np.float32)
            want = ref[rank * per:(rank + 1) * per]
            assert mine.size == want.size, (gid, rank)
            # fp32 sums of 16k products in another order (a ring all-reduce
            # of per-rank partials vs one fused accumulator): ~2e-5 apart
            assert float(np.abs(mine - want).max()) <= 5e-5 * scale, (gid, rank)
