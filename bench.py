"""Benchmark of the layout-conversion hot path (driver contract; one JSON line).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1], "1D mesh of 8: all-gather S0 -> R and
all-to-all S0R -> RS0"): one step converts a bf16 tensor S0R -> RR
(all-gather) and S0R -> RS0 (all-to-all).

  N = 1 : [65536, 8192] (1 GiB) on a mesh of 8 simulated as buffers on one
          B200, so each conversion is one collapsed exchange = one copy
          kernel over HBM (the "pack/unpack only" point of the north star).
          value = pack HBM GB/s: algorithmic bytes (every source byte read
          once + every destination byte written, i.e. the minimal HBM traffic
          of the conversion) / device time.
  N > 1 : one process per GPU (mesh [N]), weak scaling with a [8192, 8192]
          (128 MiB) S0R shard per GPU. value = bus GB/s PER GPU: the bytes a
          rank receives per step / max-over-ranks device time (NCCL busBW
          convention), roofline against the nominal 900 GB/s NVLink 5 per
          direction (the measured 770 GB/s peer copy is a second field).
          `aggregate_bus_gbs` = value x N.
  `--gpus N` without torchrun re-launches itself under
  torch.distributed.run with N ranks (127.0.0.1 rendezvous); under torchrun
  WORLD_SIZE must equal N.

Inputs are >= 128 MiB per GPU (> 126 MB L2), so no L2 flush is needed
between steps. The reference arm (--impl reference) runs the reference's own
planner (oracle/_ref: find_transform_path + conversion_cost compiled from
/root/reference) and the C oracle executing the returned steps in host RAM
with all host threads, on the SAME tensor and mesh as this arm.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "layout-conversion bus GB/s per GPU vs 900 GB/s at 2/4/8 B200; pack HBM GB/s"
SHAPE_1GPU = (65536, 8192)   # bf16, 1 GiB
SHAPE_4GIB = (262144, 8192)  # bf16, 4 GiB: the top of config 2's 1 MB - 4 GB sweep
SHARD_ROWS_NGPU = 8192       # per-GPU shard rows of [*, 8192] bf16 = 128 MiB
EB = 2
NVLINK_PEAK = 900.0          # NVLink 5, GB/s per direction per GPU (nominal, BASELINE metric)
PEER_COPY_MEASURED = 770.0   # measured peer copy per direction (B200_PROFILING.md)
CONVERSIONS = [("S0R", "RR"), ("S0R", "RS0")]


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) != 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


KERNEL_SOURCES = ["paper_2302_02599_b200/csrc/kernels/box_copy.cu",
                  "paper_2302_02599_b200/csrc/kernels/box_copy.cuh",
                  "paper_2302_02599_b200/csrc/kernels/bulk_copy.cu",
                  "paper_2302_02599_b200/csrc/runtime/runtime.cpp",
                  "paper_2302_02599_b200/csrc/runtime/plan.cpp"]


def kernel_sources_sha():
    """sha256 (16 hex) over the copy-kernel sources and the exchange compiler:
    the key under which profiles/traffic.json records ncu DRAM bytes."""
    import hashlib

    h = hashlib.sha256()
    for f in KERNEL_SOURCES:
        p = ROOT / f
        h.update(p.read_bytes() if p.exists() else b"")
    return h.hexdigest()[:16]


def stamped_traffic(key):
    """ncu dram__bytes_read+write of the dominant launch from one `ncu --set
    full` capture (tools/ncu_traffic.py writes profiles/traffic.json). Used
    only when the capture was taken from the same kernel sources as this
    build (sha stamp); otherwise null, with the reason."""
    tf = ROOT / "profiles" / "traffic.json"
    if not tf.exists():
        return None, "no ncu capture (profiles/traffic.json absent)"
    entry = json.loads(tf.read_text()).get(key)
    if not entry:
        return None, f"no ncu capture for {key}"
    sha = kernel_sources_sha()
    if entry.get("kernel_sources_sha") != sha:
        return None, f"stale ncu capture (sources {entry.get('kernel_sources_sha')} != {sha})"
    return entry["dram_bytes"], f"{entry['source']} (kernel sources {sha})"


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def workload_shape(ws):
    """The tensor this arm (and the reference arm) converts at N GPUs."""
    return SHAPE_1GPU if ws == 1 else (SHARD_ROWS_NGPU * ws, 8192)


def rank_bus_bytes(conv, ws, shard_bytes):
    """Bytes one rank receives for S0R -> `conv` on a mesh of ws (NCCL busBW
    convention: an all-gather receives (n-1) shards, an all-to-all (n-1)/n
    of one)."""
    return (ws - 1) * shard_bytes if conv == "RR" else (ws - 1) * shard_bytes // ws


def nvlink_roofline(kernel, bus_bytes, launch_ms, gpus_shared):
    achieved = bus_bytes / (launch_ms * 1e-3) / 1e9
    return {"bound": "nvlink", "kernel": kernel, "achieved": round(achieved, 1),
            "peak": NVLINK_PEAK, "peak_kind": "nominal NVLink 5 per direction per GPU",
            "unit": "GB/s", "frac": round(achieved / NVLINK_PEAK, 4),
            "frac_vs_measured_peer_copy": round(achieved / PEER_COPY_MEASURED, 4),
            "measured_peer_copy_gbs": PEER_COPY_MEASURED, "traffic": None,
            "algorithmic_bytes_per_launch": int(bus_bytes),
            "bytes_definition": "bytes this rank receives from its peers per launch",
            "launch_ms": round(launch_ms, 4),
            "note": ("ranks share one GPU: functional run, not an NVLink number"
                     if gpus_shared else "one GPU per rank")}


# ----------------------------------------------------------------------------- ours (N>1, peer)
def run_ours_peer(args):
    """N > 1 over peer memory: every rank exports its 128 MiB S0R source
    shard (CUDA IPC), maps every peer's, and each conversion is ONE pull
    kernel per rank reading its target pieces straight out of the peers'
    shards over NVLink/NVSwitch -- the collapsed pack + collective + unpack
    in a single pass -- bracketed by device-side epoch flags (no host
    barrier, no NCCL on the data path). torch.distributed (gloo) carries only
    the IPC handles, the setup barrier and the max-over-ranks timing."""
    import torch
    import torch.distributed as dist

    from paper_2302_02599_b200 import DeviceMesh, ShardingSpec, TensorMeta
    from paper_2302_02599_b200.runtime import PeerMesh, launch_count

    ws, rank, local = dist_env()
    dev_idx = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev_idx)
    dev = torch.device("cuda", dev_idx)
    dist.init_process_group("gloo")
    shape = workload_shape(ws)
    gpus_shared = torch.cuda.device_count() < ws
    meta = TensorMeta(shape, EB)
    s = ShardingSpec.parse("S0R", 1)
    pm_geo = DeviceMesh.uniform([ws])
    # Peer mapping needs P2P between the GPUs (NVLink/NVSwitch). If any rank
    # cannot map its peers, every rank agrees and the run uses NCCL instead.
    pm, err = None, ""
    try:
        pm = PeerMesh([ws], rank, dev_idx, s.per_device_bytes(meta, pm_geo))
    except Exception as e:  # noqa: BLE001
        err = f"{type(e).__name__}: {e}"
    ok = torch.tensor([0.0 if pm is None else 1.0])
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if ok.item() < 1.0:
        print(f"[bench] peer transport unavailable ({err or 'on another rank'}); using NCCL",
              file=sys.stderr, flush=True)
        if pm is not None:
            pm.close()
        dist.destroy_process_group()
        return False
    src = pm.shard(s.local_shape(meta, pm_geo), torch.bfloat16)
    gen = torch.Generator(device=dev).manual_seed(2302 + rank)
    src.view(torch.int16).random_(-32768, 32767, generator=gen)
    stream = torch.cuda.current_stream()
    in_bytes = s.per_device_bytes(meta, pm_geo)
    convs = []
    for a, b in CONVERSIONS:
        t = ShardingSpec.parse(b, 1)
        out = torch.empty(t.local_shape(meta, pm_geo), dtype=torch.bfloat16, device=dev)
        convs.append(dict(name=f"{a}->{b}", tgt=t, out=out, bus=rank_bus_bytes(b, ws, in_bytes)))
    torch.cuda.synchronize()
    dist.barrier()

    push = args.transport == "push"

    def xchg(c):
        """One exchange of the peer transport: the fused pull (default) or the
        push form (remote stores into the receivers' exported outputs)."""
        if push:
            return pm.push_async(s, c["tgt"], meta, src, stream=stream)
        pm.exchange_async(s, c["tgt"], meta, c["out"], stream=stream)
        return c["out"]

    def step():
        for c in convs:
            xchg(c)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps * len(convs))]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = launch_count()
    with ClockSampler(dev_idx) as clk:
        t0.record(stream)
        k = 0
        for _ in range(args.steps):
            for c in convs:
                evs[k][0].record(stream)
                xchg(c)
                evs[k][1].record(stream)
                k += 1
        t1.record(stream)
        torch.cuda.synchronize()
    launches = launch_count() - launches0
    per = {c["name"]: [] for c in convs}
    for i, (a_, b_) in enumerate(evs):
        per[convs[i % len(convs)]["name"]].append(a_.elapsed_time(b_))
    v = torch.tensor([t0.elapsed_time(t1)] + [statistics.mean(per[c["name"]]) for c in convs],
                     dtype=torch.float64)
    dist.all_reduce(v, op=dist.ReduceOp.MAX)
    ms_per_step = float(v[0]) / args.steps
    per_ms = {c["name"]: float(v[1 + i]) for i, c in enumerate(convs)}
    step_bus = sum(c["bus"] for c in convs)  # per rank (every rank receives the same)
    value = step_bus / (ms_per_step * 1e-3) / 1e9
    dom = max(convs, key=lambda c: per_ms[c["name"]])
    roof = nvlink_roofline(f"box_copy {'push' if push else 'pull'} kernel over peer pointers ({dom['name']})",
                           dom["bus"], per_ms[dom["name"]], gpus_shared)
    # e2e through the public API with host buffers: H2D of this rank's source
    # shard (after the readers of the last epoch finished), both exchanges,
    # D2H of both converted shards -- every step, one stream.
    host_in = torch.empty(src.shape, dtype=src.dtype).pin_memory()
    host_in.copy_(src)
    host_out = [torch.empty(c["out"].shape, dtype=c["out"].dtype).pin_memory() for c in convs]
    e_steps = max(4, min(args.steps, 8))

    def e2e_step():
        pm.wait_readers(stream=stream)
        src.copy_(host_in, non_blocking=True)
        for c, h in zip(convs, host_out):
            h.copy_(xchg(c).view(c["out"].dtype).view(c["out"].shape), non_blocking=True)

    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize()
    dist.barrier()
    ea, ez = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ea.record(stream)
    for _ in range(e_steps):
        e2e_step()
    ez.record(stream)
    torch.cuda.synchronize()
    et = torch.tensor([ea.elapsed_time(ez) / e_steps], dtype=torch.float64)
    dist.all_reduce(et, op=dist.ReduceOp.MAX)
    e2e = {"value": round(step_bus / (float(et[0]) * 1e-3) / 1e9, 2), "unit": "GB/s per GPU",
           "h2d_bytes_per_step": in_bytes,
           "d2h_bytes_per_step": sum(h.numel() * h.element_size() for h in host_out),
           "ms_per_step": round(float(et[0]), 3), "steps": e_steps,
           "note": "per rank: pinned H2D of its source shard, both exchanges, D2H of both "
                   "converted shards; one stream; max over ranks"}
    result = {
        "metric": METRIC, "value": round(value, 1), "unit": "GB/s per GPU", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (random bf16 bit patterns, torch.random_ on device)",
        "aggregate_bus_gbs": round(value * ws, 1), "bus_bytes_per_rank_per_step": int(step_bus),
        "config": {"workload": "configs[1]: mesh of N, S0R->RR all-gather + S0R->RS0 all-to-all",
                   "tensor": list(shape), "mesh": [ws], "transport": "push" if push else "peer",
                   "gpus_shared": gpus_shared,
                   "mode": ("one process per GPU, push kernel (remote stores) over peer memory, "
                            "device-side epoch flags" if push else
                            "one process per GPU, fused pull kernel over peer memory, "
                            "device-side epoch flags"),
                   "path": "collapsed exchange (one %s kernel per rank)" % ("push" if push else "pull"),
                   "l2": "per-GPU shard 128 MiB > L2", "parallelism": f"mesh[{ws}]"},
        "per_conversion_ms": {k: round(v_, 4) for k, v_ in per_ms.items()},
        "roofline": roof, "gpu_launches": int(launches), "clocks": clk.summary(), "e2e": e2e,
    }
    torch.cuda.synchronize()
    dist.barrier()
    pm.close()
    if not args.no_sweep:
        result["mesh_sweep"] = peer_mesh_sweep(ws, rank, dev_idx)
    if rank == 0:
        print(json.dumps(result))
    dist.destroy_process_group()
    return True


def peer_mesh_sweep(ws, rank, dev_idx, iters=10):
    """configs 3/4 on the real 2-D / 3-D meshes ([2,2] at N=4; [2,4] and
    [2,2,2] at N=8) over the peer transport: bus GB/s per GPU = max over ranks
    of the bytes a rank pulls / max-over-ranks time per exchange (flags
    included), vs the nominal 900 GB/s (and the measured 770 GB/s peer copy)."""
    import torch
    import torch.distributed as dist

    from paper_2302_02599_b200 import DeviceMesh, ShardingSpec, TensorMeta
    from paper_2302_02599_b200.runtime import PeerMesh

    meshes = {4: [[2, 2]], 8: [[2, 4], [2, 2, 2]]}.get(ws, [])
    stream = torch.cuda.current_stream()
    rows = []
    for ms in meshes:
        cases = _sweep_cases(ms)
        geo = DeviceMesh.uniform(ms)
        biggest = max(ShardingSpec.parse(a, len(ms)).per_device_bytes(TensorMeta(sh, 2), geo)
                      for sh, a, _ in cases)
        pm = PeerMesh(ms, rank, dev_idx, biggest)
        for shape, a, b in cases:
            meta = TensorMeta(shape, 2)
            s, t = ShardingSpec.parse(a, len(ms)), ShardingSpec.parse(b, len(ms))
            out = torch.empty(t.local_shape(meta, pm.geo), dtype=torch.bfloat16,
                              device=f"cuda:{dev_idx}")
            wire = pm.exchange_traffic(s, t, meta)["wire_in"]
            for _ in range(2):
                pm.exchange_async(s, t, meta, out, stream=stream)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(iters):
                pm.exchange_async(s, t, meta, out, stream=stream)
            e1.record(stream)
            torch.cuda.synchronize()
            v = torch.tensor([e0.elapsed_time(e1) / iters, float(wire)], dtype=torch.float64)
            dist.all_reduce(v, op=dist.ReduceOp.MAX)
            ms_t, wire = float(v[0]), float(v[1])
            rows.append({"mesh": ms, "tensor": list(shape), "conversion": f"{a}->{b}",
                         "us": round(ms_t * 1e3, 2), "bus_bytes": int(wire),
                         "bus_gbs": round(wire / ms_t / 1e6, 1) if wire else None,
                         "frac": round(wire / ms_t / 1e6 / NVLINK_PEAK, 3) if wire else None,
                         "frac_vs_measured_peer_copy":
                             round(wire / ms_t / 1e6 / PEER_COPY_MEASURED, 3) if wire else None})
            del out
        torch.cuda.synchronize()
        dist.barrier()
        pm.close()
    fr = [r["frac"] for r in rows if r.get("frac") is not None]
    return {"rows": rows, "frac_min": min(fr) if fr else None,
            "frac_median": statistics.median(fr) if fr else None, "peak": NVLINK_PEAK,
            "kind": "bus GB/s per GPU (bytes pulled over peer memory), transport peer"}


# ----------------------------------------------------------------------------- ours
def run_ours(args):
    import numpy as np
    import torch

    from paper_2302_02599_b200 import ShardingSpec, TensorMeta, find_transform_path
    from paper_2302_02599_b200.runtime import Mesh, launch_count

    ws, rank, local = dist_env()
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        import torch.distributed as dist

        if torch.cuda.device_count() < ws:
            # ranks share a GPU (functional run): NCCL refuses two ranks of one
            # host on one device, so each rank poses as its own host and NCCL
            # connects them over sockets on loopback (tests/test_gpu_nccl.py)
            os.environ.setdefault("NCCL_HOSTID", f"apl-bench-host-{rank}")
            os.environ.setdefault("NCCL_SOCKET_IFNAME", "lo")
            os.environ.setdefault("NCCL_IB_DISABLE", "1")
        dist.init_process_group("nccl", device_id=dev)
        mesh = Mesh.from_process_group([ws])
        shape = workload_shape(ws)
        ndev = ws
    else:
        mesh = Mesh.local([8], device=local)
        shape = SHAPE_1GPU
        ndev = 8
    meta = TensorMeta(shape, EB)
    geo = mesh.geo
    stream = torch.cuda.current_stream()

    convs, sources = [], {}
    for a, b in CONVERSIONS:
        s, t = ShardingSpec.parse(a, 1), ShardingSpec.parse(b, 1)
        path = find_transform_path(s, t, geo, meta)
        if a not in sources:  # both conversions read the same S0R tensor
            ins = [torch.empty(s.local_shape(meta, geo), dtype=torch.bfloat16, device=dev)
                   for _ in range(mesh.num_local)]
            gen = torch.Generator(device=dev).manual_seed(2302 + rank)
            for x in ins:  # synthetic payload, generated on device (bytes are moved, not interpreted)
                x.view(torch.int16).random_(-32768, 32767, generator=gen)
            sources[a] = ins
        ins = sources[a]
        outs = [torch.empty(t.local_shape(meta, geo), dtype=torch.bfloat16, device=dev)
                for _ in range(mesh.num_local)]
        out_bytes = t.per_device_bytes(meta, geo)
        in_bytes = s.per_device_bytes(meta, geo)
        # algorithmic HBM bytes per launch on the local devices: every source
        # byte read once + every destination byte written (library accounting
        # of the compiled exchange, identical to what the kernel moves)
        traffic = mesh.exchange_traffic(s, t, meta)
        hbm = traffic["hbm_read"] + traffic["hbm_write"]
        bus = rank_bus_bytes(b, ndev, in_bytes)  # bytes each rank receives
        engine = mesh.exchange_engine(s, t, meta)
        conv = mesh.prepare(path, meta, fuse=True)  # public API: compiled once, launched per step
        convs.append(dict(name=f"{a}->{b}", path=path, conv=conv, ins=ins, outs=outs, hbm=hbm, bus=bus,
                          in_bytes=in_bytes, out_bytes=out_bytes,
                          kernel="bulk_copy_kernel (TMA cp.async.bulk ring)" if engine == "bulk"
                          else "box_copy_kernel<16,U,NO,MINB> (LDG/STG.128)"))

    def step():
        for c in convs:
            c["conv"](c["ins"], c["outs"], stream=stream)

    def barrier():
        if ws > 1:
            import torch.distributed as dist

            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()

    # per-conversion kernel timing (events on the launching stream)
    n_ev = args.steps * len(convs)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(n_ev)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = launch_count()
    with ClockSampler(local) as clk:
        barrier()
        t0.record(stream)
        k = 0
        for _ in range(args.steps):
            for c in convs:
                evs[k][0].record(stream)
                c["conv"](c["ins"], c["outs"], stream=stream)
                evs[k][1].record(stream)
                k += 1
        t1.record(stream)
        barrier()
    launches = launch_count() - launches0
    total_ms = t0.elapsed_time(t1)
    per_conv_ms = {c["name"]: [] for c in convs}
    for i in range(n_ev):
        per_conv_ms[convs[i % len(convs)]["name"]].append(evs[i][0].elapsed_time(evs[i][1]))
    if ws > 1:
        import torch.distributed as dist

        tt = torch.tensor([total_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())

    ms_per_step = total_ms / args.steps
    hbm_peak, peak_kind = peaks()
    if ws == 1:
        step_bytes = sum(c["hbm"] for c in convs)
        unit = "GB/s"
    else:  # per-GPU bus bytes (every rank receives the same)
        step_bytes = sum(c["bus"] for c in convs)
        unit = "GB/s per GPU"
    value = step_bytes / (ms_per_step * 1e-3) / 1e9

    # roofline of the dominant kernel (the box-copy of S0R->RR, largest share)
    dom = max(convs, key=lambda c: statistics.mean(per_conv_ms[c["name"]]))
    dom_ms = statistics.mean(per_conv_ms[dom["name"]])
    if ws == 1:
        traffic, traffic_src = stamped_traffic(f"n1:{dom['name']}")
        achieved = dom["hbm"] / (dom_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "kernel": f"{dom['kernel']} ({dom['name']}, 8 simulated devices)",
                "achieved": round(achieved, 1), "peak": hbm_peak, "peak_kind": peak_kind,
                "unit": "GB/s", "frac": round(achieved / hbm_peak, 4), "traffic": traffic,
                "traffic_source": traffic_src,
                "algorithmic_bytes_per_launch": dom["hbm"],
                "bytes_definition": "source bytes read once + destination bytes written",
                "launch_ms": round(dom_ms, 4)}
    else:
        roof = nvlink_roofline(f"{dom['name']} exchange (NCCL collective + box_copy pack/unpack)",
                               dom["bus"], dom_ms, torch.cuda.device_count() < ws)

    result = {
        "metric": METRIC, "value": round(value, 1), "unit": unit, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (random bf16 bit patterns, torch.random_ on device)",
        "config": {"workload": f"configs[1]: mesh of {ndev}, S0R->RR all-gather + S0R->RS0 "
                               "all-to-all",
                   "tensor": list(shape), "mesh": [ndev],
                   "mode": "simulated 8-device mesh on 1 GPU (pack/unpack only)" if ws == 1
                   else "one process per GPU, NCCL per mesh-axis communicator",
                   "transport": "simulated" if ws == 1 else "nccl",
                   "path": "collapsed exchange (APL_FUSE_CHAIN)",
                   "l2": "inputs 1 GiB > 126 MB L2, no flush needed" if ws == 1 else
                   "per-GPU shard 128 MiB > L2",
                   "parallelism": f"mesh[{ndev}]"},
        "per_conversion_ms": {k: round(statistics.mean(v), 4) for k, v in per_conv_ms.items()},
        "roofline": roof,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if ws > 1:
        result["aggregate_bus_gbs"] = round(value * ws, 1)
    result["e2e"] = run_e2e(args, mesh, meta, convs, stream, ws)
    if not args.no_sweep:
        result["mesh_sweep"] = mesh_sweep(ws, rank, dev, stream, hbm_peak)
        if ws == 1:
            result["config2_4gib"] = size_point(args, SHAPE_4GIB, dev, hbm_peak)
    if ws == 1 and not args.no_cpu:
        result["cpu_baseline"] = cpu_baseline(args)
    if rank == 0:
        print(json.dumps(result))
    if ws > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def _distinct_shards(spec, geo, meta):
    """Device indices holding distinct blocks under `spec` (replicas of one
    block are bit-identical by construction and read back once)."""
    seen, keep = set(), []
    for d in range(geo.num_devices()):
        coord = geo.coord_of(d)
        key = []
        for dim in spec.dims:
            s = 0
            for a in dim.axes:
                s = s * geo.shape[a] + coord[a]
            key.append(s)
        if tuple(key) not in seen:
            seen.add(tuple(key))
            keep.append(d)
    return keep


def run_e2e(args, mesh, meta, convs, stream, ws=1):
    """Same metric through the public API with HOST buffers. Every step:
    pinned H2D of the step's input shards, the conversions (prepared
    conversions, the public API), D2H of the converted result (each distinct
    target shard once). The three legs run on their own streams and device
    shards are double-buffered, so step i's D2H overlaps step i+1's H2D and
    conversions (PCIe is full duplex)."""
    import torch

    from paper_2302_02599_b200 import ShardingSpec

    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    # distinct input tensors (conversions of the same tensor share its H2D)
    srcs = []
    for c in convs:
        if not any(c["ins"] is x for x in srcs):
            srcs.append(c["ins"])
    src_of = [next(i for i, x in enumerate(srcs) if c["ins"] is x) for c in convs]
    sets = []  # per buffer set: (input lists, output lists)
    for b in range(2):
        ins_b = srcs if b == 0 else [[torch.empty_like(x) for x in lst] for lst in srcs]
        outs_b = [c["outs"] if b == 0 else [torch.empty_like(x) for x in c["outs"]] for c in convs]
        sets.append((ins_b, outs_b))
    host_in = [[torch.empty_like(x, device="cpu").pin_memory() for x in lst] for lst in srcs]
    for lst, hi in zip(srcs, host_in):
        for h, x in zip(hi, lst):
            h.copy_(x)
    keep = []
    for c in convs:
        a, b = c["name"].split("->")
        if mesh.distributed:  # every rank reads back its own converted shard
            keep.append([0])
        else:
            keep.append(_distinct_shards(ShardingSpec.parse(b, mesh.geo.rank()), mesh.geo, meta))
    host_out = [[torch.empty_like(c["outs"][d], device="cpu").pin_memory() for d in k]
                for c, k in zip(convs, keep)]
    h2d = sum(x.numel() * x.element_size() for hi in host_in for x in hi)
    d2h = sum(x.numel() * x.element_size() for ho in host_out for x in ho)
    steps = max(4, min(args.steps, 8))
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_cmp = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]

    def e2e_step(i):
        b = i % 2
        ins_b, outs_b = sets[b]
        with torch.cuda.stream(s_in):
            if i >= 2:
                s_in.wait_event(ev_cmp[b])           # step i-2 finished reading set b
            for lst, hi in zip(ins_b, host_in):
                for x, h in zip(lst, hi):
                    x.copy_(h, non_blocking=True)
            ev_in[b].record(s_in)
        stream.wait_event(ev_in[b])
        if i >= 2:
            stream.wait_event(ev_out[b])             # step i-2's D2H drained set b
        for c, k, outs in zip(convs, src_of, outs_b):
            c["conv"](ins_b[k], outs, stream=stream)
        ev_cmp[b].record(stream)
        with torch.cuda.stream(s_out):
            s_out.wait_event(ev_cmp[b])
            for outs, ho, kk in zip(outs_b, host_out, keep):
                for h, d in zip(ho, kk):
                    h.copy_(outs[d], non_blocking=True)
            ev_out[b].record(s_out)

    for i in range(2):
        e2e_step(i)
    torch.cuda.synchronize()
    a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s_in)
    for i in range(steps):
        e2e_step(i)
    s_out.wait_stream(s_in)
    s_out.wait_stream(stream)
    z.record(s_out)
    torch.cuda.synchronize()
    ms = a.elapsed_time(z) / steps
    if ws > 1:
        import torch.distributed as dist

        t = torch.tensor([ms], device=f"cuda:{mesh.device}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        step_bytes = sum(c["bus"] for c in convs)  # per GPU, the same metric as `value`
    else:
        step_bytes = sum(c["hbm"] for c in convs)
    return {"value": round(step_bytes / (ms * 1e-3) / 1e9, 2),
            "unit": "GB/s" if ws == 1 else "GB/s per GPU",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": round(ms, 3),
            "steps": steps,
            "note": "pinned H2D of the input tensor's shards (once: both conversions read the "
                    "same tensor) + D2H of every distinct converted shard (replicas of an RR "
                    "block read once), 3 streams, double-buffered shards"}


# ----------------------------------------------------------------------------- configs 3/4
CONFIG3_SPECS = ["S01R", "S0S1", "S1S0", "RS01", "RR"]


def _sweep_cases(mesh_shape):
    """BASELINE configs 3/4 conversions for a mesh: every ordered pair among
    the config-3 specs on [8192, 8192] bf16 (2x4; the same specs on 2x2), and
    the config-4 chains on 2x2x2."""
    if len(mesh_shape) == 2:
        return [((8192, 8192), a, b) for a in CONFIG3_SPECS for b in CONFIG3_SPECS if a != b]
    return [((8192, 8192), "S012R", "RS012"), ((8192, 8192), "RS012", "S012R"),
            ((512, 512, 256), "S0S1R", "RS1S0"), ((512, 512, 256), "RS1S0", "S0S1R")]


def mesh_sweep(ws, rank, dev, stream, hbm_peak, iters=20):
    """configs 3/4 (2-D / 3-D meshes) through the same public API.
    N = 1: 2x4 and 2x2x2 simulated on one GPU -> pack HBM GB/s vs the
    measured copy peak. N = 4 / 8: the real meshes ([2,2]; [2,4] and [2,2,2])
    over NCCL -> bus GB/s per GPU = max over ranks of the minimal one-shot
    bytes a rank receives / max-over-ranks time, vs the
    nominal 900 GB/s NVLink (and the measured 770 GB/s peer copy). Collapsed
    exchanges, events on the launch
    stream."""
    import torch

    from paper_2302_02599_b200 import ShardingSpec, TensorMeta, find_transform_path
    from paper_2302_02599_b200.runtime import Mesh

    meshes = {1: [[2, 4], [2, 2, 2]], 4: [[2, 2]], 8: [[2, 4], [2, 2, 2]]}.get(ws, [])
    rows = []
    for ms in meshes:
        mesh = Mesh.local(ms, device=dev.index or 0) if ws == 1 else Mesh.from_process_group(ms)
        for shape, a, b in _sweep_cases(ms):
            meta = TensorMeta(shape, 2)
            s, t = ShardingSpec.parse(a, len(ms)), ShardingSpec.parse(b, len(ms))
            path = find_transform_path(s, t, mesh.geo, meta)
            ins = [torch.empty(s.local_shape(meta, mesh.geo), dtype=torch.bfloat16, device=dev)
                   for _ in range(mesh.num_local)]
            outs = [torch.empty(t.local_shape(meta, mesh.geo), dtype=torch.bfloat16, device=dev)
                    for _ in range(mesh.num_local)]
            conv = mesh.prepare(path, meta, fuse=True)
            tr = mesh.exchange_traffic(s, t, meta)
            for _ in range(3):
                conv(ins, outs, stream=stream)
            if ws > 1:
                import torch.distributed as dist

                dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(iters):
                conv(ins, outs, stream=stream)
            e1.record(stream)
            torch.cuda.synchronize()
            ms_t = e0.elapsed_time(e1) / iters
            row = {"mesh": ms, "tensor": list(shape), "conversion": f"{a}->{b}",
                   "ref_steps": len(path.steps), "us": None}
            if ws == 1:
                nbytes = tr["hbm_read"] + tr["hbm_write"]
                row.update(us=round(ms_t * 1e3, 2), hbm_bytes=nbytes,
                           gbs=round(nbytes / ms_t / 1e6, 1),
                           frac=round(nbytes / ms_t / 1e6 / hbm_peak, 3))
            else:
                import torch.distributed as dist

                v = torch.tensor([ms_t, float(tr["wire_in"])], device=dev, dtype=torch.float64)
                dist.all_reduce(v, op=dist.ReduceOp.MAX)
                ms_t, wire = float(v[0]), float(v[1])
                row.update(us=round(ms_t * 1e3, 2), bus_bytes=int(wire),
                           bus_gbs=round(wire / ms_t / 1e6, 1) if wire else None,
                           frac=round(wire / ms_t / 1e6 / NVLINK_PEAK, 3) if wire else None,
                           frac_vs_measured_peer_copy=round(
                               wire / ms_t / 1e6 / PEER_COPY_MEASURED, 3) if wire else None)
            rows.append(row)
            conv.close()
            del ins, outs
        mesh.close()
        torch.cuda.empty_cache()
    fr = [r["frac"] for r in rows if r.get("frac") is not None]
    return {"rows": rows, "frac_min": min(fr) if fr else None,
            "frac_median": statistics.median(fr) if fr else None,
            "peak": hbm_peak if ws == 1 else NVLINK_PEAK,
            "kind": "pack HBM GB/s (simulated mesh)" if ws == 1 else
                    "bus GB/s per GPU (minimal one-shot bytes, NCCL)"}


# ----------------------------------------------------------------------------- CPU legs
def cpu_model():
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


class CpuWorkload:
    """The reference CPU path of one step on host RAM: the reference planner
    (oracle/_ref find_transform_path, compiled from /root/reference) picks each
    conversion's steps, the C oracle executes them on the N simulated devices.
    Source shards and destination buffers are allocated once (reused every
    step, as the GPU arm's are), so a step times the byte movement."""

    def __init__(self, ndev, shape):
        from oracle import data as O
        from oracle import ref as R

        self.O, self.R = O, R
        self.ndev, self.shape = ndev, tuple(shape)
        g = O.fill_global(self.shape, EB)
        self.ins = O.shards(g, O.parse_spec("S0R", 1), [ndev])
        del g
        self.outs = {}
        for _, b in CONVERSIONS:
            dims = O.parse_spec(b, 1)
            ls = O.local_shape(self.shape, dims, [ndev])
            self.outs[b] = [O.np.empty(ls, dtype=self.ins[0].dtype) for _ in range(ndev)]
            for o in self.outs[b]:
                o.fill(0)  # first touch outside the timed steps
        self.in_bytes = sum(x.nbytes for x in self.ins)

    def step(self, threads):
        """-> (seconds, algorithmic bytes, per-GPU bus bytes)."""
        O, R = self.O, self.R
        O.set_threads(threads)
        total_s, total_b, bus = 0.0, 0, 0
        for a, b in CONVERSIONS:
            t0 = time.perf_counter()
            if R.available():
                rc, steps, _ = R.find_path([self.ndev], list(self.shape), EB, a, b)
                assert rc == 0, steps
            else:
                steps = [(0, 0, -1, 0, "R")] if b == "RR" else [(3, 0, 1, 0, "RS0")]
            O.replay(self.shape, O.parse_spec(a, 1), [self.ndev], steps, self.ins,
                     outs=self.outs[b])
            total_s += time.perf_counter() - t0
            # same accounting as the GPU arm: source bytes read once + bytes written
            total_b += self.in_bytes + sum(o.nbytes for o in self.outs[b])
            bus += rank_bus_bytes(b, self.ndev, self.ins[0].nbytes)
        return total_s, total_b, bus


def cpu_baseline(args):
    """The reference CPU path on the SAME [65536, 8192] tensor and mesh [8] as
    the GPU arm, all host threads, bounded to ~10 s; plus one single-thread
    step."""
    threads = os.cpu_count() or 1
    w = CpuWorkload(8, SHAPE_1GPU)
    w.step(threads)  # warm-up
    secs, nbytes, reps = 0.0, 0, 0
    while secs < 10.0 and reps < 20:
        s_, b, _ = w.step(threads)
        secs += s_
        nbytes += b
        reps += 1
    s1, b1, _ = w.step(1)
    return {"value": round(nbytes / secs / 1e9, 3), "unit": "GB/s", "cores": threads,
            "kind": "reference" if _ref_available() else "port",
            "single_thread": {"value": round(b1 / s1 / 1e9, 3), "unit": "GB/s", "cores": 1,
                              "ms_per_step": round(1e3 * s1, 1)},
            "cpu_model": cpu_model(),
            "sample": f"{reps} full steps (S0R->RR + S0R->RS0 of the same [{SHAPE_1GPU[0]},"
                      f"{SHAPE_1GPU[1]}] bf16 tensor, mesh [8] simulated in host RAM); path "
                      f"from the reference planner ("
                      f"{'oracle/_ref' if _ref_available() else 'n/a'}), bytes moved by the C "
                      f"oracle with {threads} threads; same algorithmic-byte accounting as "
                      f"the GPU arm"}


def _ref_available():
    from oracle import ref as R

    return R.available()


def planner_timings(iters=2000):
    """Reference planner (oracle/_ref) per BASELINE config 1-4: mean us per
    uncached find_transform_path + conversion_cost, and per cached
    PathCache::get hit (layout.cpp:331-346)."""
    if not _ref_available():
        return None
    from oracle import ref as R

    cases = [
        (1, [2, 2], [1024, 1024], 4, [("S0R", "RS0")]),
        (2, [8], list(SHAPE_1GPU), 2, list(CONVERSIONS)),
        (3, [2, 4], [8192, 8192], 2,
         [(a, b) for a in CONFIG3_SPECS for b in CONFIG3_SPECS if a != b]),
        (4, [2, 2, 2], [8192, 8192], 2, [("S012R", "RS012"), ("RS012", "S012R")]),
        (4, [2, 2, 2], [512, 512, 256], 2, [("S0S1R", "RS1S0"), ("RS1S0", "S0S1R")]),
    ]
    out = []
    for cfg, mesh, shape, eb, pairs in cases:
        miss = [R.time_paths(mesh, shape, eb, a, b, iters, hits=False) for a, b in pairs]
        hit = [R.time_paths(mesh, shape, eb, a, b, iters * 10, hits=True) for a, b in pairs]
        out.append({"config": cfg, "mesh": mesh, "tensor": shape, "pairs": len(pairs),
                    "search_us_mean": round(1e6 * statistics.mean(miss), 3),
                    "search_us_max": round(1e6 * max(miss), 3),
                    "cache_hit_us_mean": round(1e6 * statistics.mean(hit), 4)})
    return out


def run_reference(args):
    """--impl reference: the reference's CPU path (reference planner + C
    oracle byte movement) on this arm's config at N: tensor and mesh are
    exactly the GPU arm's (`workload_shape`), so the two lines are like for
    like. At N > 1 the value is per-GPU bus GB/s (bytes one simulated device
    receives / step time), the GPU arm's N > 1 metric."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    n = max(ws, args.gpus)
    ndev = 8 if n == 1 else n
    shape = workload_shape(n)
    threads = os.cpu_count() or 1
    w = CpuWorkload(ndev, shape)
    for _ in range(args.warmup):
        w.step(threads)
    secs, nbytes, bus = 0.0, 0, 0
    for _ in range(args.steps):
        s_, b, bb = w.step(threads)
        secs += s_
        nbytes += b
        bus += bb
    value = (nbytes if n == 1 else bus) / secs / 1e9
    unit = "GB/s" if n == 1 else "GB/s per GPU"
    s1, b1, bb1 = w.step(1)
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": unit, "n_gpus": n,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * secs / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (splitmix64 bit patterns, oracle_fill)",
        "impl": "reference",
        "config": {"workload": f"configs[1]: mesh of {ndev}, S0R->RR all-gather + S0R->RS0 "
                               "all-to-all",
                   "tensor": list(shape), "mesh": [ndev],
                   "mode": "host RAM, all host threads", "parallelism": "cpu"},
        "cpu_baseline": {"value": round(value, 3), "unit": unit, "cores": threads,
                         "kind": "reference" if _ref_available() else "port",
                         "cpu_model": cpu_model(),
                         "single_thread": {"value": round((b1 if n == 1 else bb1) / s1 / 1e9, 3),
                                           "unit": unit, "cores": 1,
                                           "ms_per_step": round(1e3 * s1, 1)},
                         "sample": f"per step: S0R->RR + S0R->RS0 of the full "
                                   f"[{shape[0]},{shape[1]}] bf16 tensor on {ndev} simulated "
                                   "devices (the GPU arm's exact workload); the reference "
                                   "planner (oracle/_ref) picks the path, the C oracle moves "
                                   "the bytes"},
        "planner": planner_timings(),
        "e2e": {"value": round(value, 3), "unit": unit, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def size_point(args, shape, dev, hbm_peak, iters=10):
    """One extra config-2 size on the simulated mesh of 8 (e.g. the sweep's
    4 GiB top): S0R->RR + S0R->RS0, device time per step, pack HBM GB/s."""
    import torch

    from paper_2302_02599_b200 import ShardingSpec, TensorMeta, find_transform_path
    from paper_2302_02599_b200.runtime import Mesh

    mesh = Mesh.local([8], device=dev.index or 0)
    meta = TensorMeta(shape, EB)
    s = ShardingSpec.parse("S0R", 1)
    ins = [torch.empty(s.local_shape(meta, mesh.geo), dtype=torch.bfloat16, device=dev)
           for _ in range(8)]
    for x in ins:
        x.view(torch.int16).random_(-32768, 32767)
    stream = torch.cuda.current_stream()
    rows, total_b, total_ms = [], 0, 0.0
    for a, b in CONVERSIONS:
        t = ShardingSpec.parse(b, 1)
        outs = [torch.empty(t.local_shape(meta, mesh.geo), dtype=torch.bfloat16, device=dev)
                for _ in range(8)]
        conv = mesh.prepare(find_transform_path(s, t, mesh.geo, meta), meta, fuse=True)
        tr = mesh.exchange_traffic(s, t, meta)
        nbytes = tr["hbm_read"] + tr["hbm_write"]
        for _ in range(3):
            conv(ins, outs, stream=stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(iters):
            conv(ins, outs, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / iters
        rows.append({"conversion": f"{a}->{b}", "ms": round(ms, 4), "hbm_bytes": nbytes,
                     "gbs": round(nbytes / ms / 1e6, 1),
                     "frac": round(nbytes / ms / 1e6 / hbm_peak, 4)})
        total_b += nbytes
        total_ms += ms
        conv.close()
        del outs
        torch.cuda.empty_cache()
    mesh.close()
    del ins
    torch.cuda.empty_cache()
    return {"tensor": list(shape), "mesh": [8], "ms_per_step": round(total_ms, 4),
            "value": round(total_b / total_ms / 1e6, 1), "unit": "GB/s",
            "frac": round(total_b / total_ms / 1e6 / hbm_peak, 4), "per_conversion": rows}


def spawn(args):
    """`--gpus N` outside torchrun: re-launch this script as N ranks under
    torch.distributed.run (one process per GPU, 127.0.0.1 rendezvous) and
    pass rank 0's line through."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-sweep", action="store_true", help="skip the configs 3/4 mesh sweep")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--transport", default="peer", choices=["peer", "push", "nccl"],
                    help="N > 1: fused peer-memory pull (default), peer-memory push (remote "
                         "stores), or NCCL per mesh-axis communicator + pack/unpack kernels")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    ws = dist_env()[0]
    if "WORLD_SIZE" in os.environ and ws != args.gpus:
        sys.exit(f"bench.py: WORLD_SIZE={ws} but --gpus {args.gpus}")
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn(args))
    if ws > 1 and args.transport in ("peer", "push"):
        if not run_ours_peer(args):
            run_ours(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
