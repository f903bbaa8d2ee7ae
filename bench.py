"""Benchmark of the layout-conversion hot path (driver contract; one JSON line).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1], "1D mesh of 8: all-gather S0 -> R and
all-to-all S0R -> RS0"): one step converts a [65536, 8192] bf16 tensor
(1 GiB) S0R -> RR (all-gather) and S0R -> RS0 (all-to-all) on a mesh of 8.

  N = 1 : the 8 mesh devices are simulated as buffers on one B200, so each
          conversion is one collapsed exchange = one box-copy kernel over HBM
          (the "pack/unpack only" point of the north star). value = pack HBM
          GB/s: algorithmic bytes (every source byte read once + every
          destination byte written, i.e. the minimal HBM traffic of the
          conversion) / device time.
  N > 1 : one process per GPU over NCCL (mesh [N]), weak scaling with a
          128 MiB shard per GPU; value = bus bytes received by all ranks /
          max-over-ranks device time (aggregate bus GB/s).

Inputs are 1 GiB (> 126 MB L2), so no L2 flush is needed between steps.
The reference arm (--impl reference) runs the reference's own planner
(oracle/_ref: find_transform_path + conversion_cost compiled from
/root/reference) and the C oracle executing the returned steps in host RAM
with all host threads, on a bounded sample of the same workload.
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
SHARD_ROWS_NGPU = 8192       # per-GPU shard rows of [*, 8192] bf16 = 128 MiB
EB = 2
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


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


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
    shape = (SHARD_ROWS_NGPU * ws, 8192)
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
        bus = (ws - 1) * in_bytes if b == "RR" else (ws - 1) * in_bytes // ws
        convs.append(dict(name=f"{a}->{b}", tgt=t, out=out, bus=bus))
    torch.cuda.synchronize()
    dist.barrier()

    def step():
        for c in convs:
            pm.exchange_async(s, c["tgt"], meta, c["out"], stream=stream)

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
                pm.exchange_async(s, c["tgt"], meta, c["out"], stream=stream)
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
    step_bus = sum(c["bus"] for c in convs) * ws
    value = step_bus / (ms_per_step * 1e-3) / 1e9
    dom = max(convs, key=lambda c: per_ms[c["name"]])
    achieved = dom["bus"] / (per_ms[dom["name"]] * 1e-3) / 1e9
    roof = {"bound": "nvlink", "kernel": f"box_copy/bulk pull kernel over peer pointers ({dom['name']})",
            "achieved": round(achieved, 1), "peak": 770.0,
            "peak_kind": "measured peer copy per direction per GPU (B200_PROFILING.md)",
            "unit": "GB/s", "frac": round(achieved / 770.0, 4), "traffic": None,
            "algorithmic_bytes_per_launch": dom["bus"],
            "bytes_definition": "bytes this rank receives over NVLink (NCCL busBW convention)",
            "launch_ms": round(per_ms[dom["name"]], 4)}
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
            pm.exchange_async(s, c["tgt"], meta, c["out"], stream=stream)
            h.copy_(c["out"], non_blocking=True)

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
    e2e = {"value": round(step_bus / (float(et[0]) * 1e-3) / 1e9, 2), "unit": "GB/s",
           "h2d_bytes_per_step": in_bytes,
           "d2h_bytes_per_step": sum(h.numel() * h.element_size() for h in host_out),
           "ms_per_step": round(float(et[0]), 3), "steps": e_steps,
           "note": "per rank: pinned H2D of its source shard, both exchanges, D2H of both "
                   "converted shards; one stream; max over ranks"}
    result = {
        "metric": METRIC, "value": round(value, 1), "unit": "GB/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (random bf16 bit patterns generated on device)",
        "config": {"workload": "configs[1]: mesh of N, S0R->RR all-gather + S0R->RS0 all-to-all",
                   "tensor": list(shape), "mesh": [ws], "transport": "peer",
                   "mode": "one process per GPU, fused pull kernel over peer memory, "
                           "device-side epoch flags",
                   "path": "collapsed exchange (one pull kernel per rank)",
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
    included), vs the measured 770 GB/s peer copy."""
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
                         "frac": round(wire / ms_t / 1e6 / 770.0, 3) if wire else None})
            del out
        torch.cuda.synchronize()
        dist.barrier()
        pm.close()
    fr = [r["frac"] for r in rows if r.get("frac") is not None]
    return {"rows": rows, "frac_min": min(fr) if fr else None,
            "frac_median": statistics.median(fr) if fr else None, "peak": 770.0,
            "kind": "bus GB/s per GPU (bytes pulled over peer memory), transport peer"}


# ----------------------------------------------------------------------------- ours
def run_ours(args):
    import numpy as np
    import torch

    from paper_2302_02599_b200 import ShardingSpec, TensorMeta, find_transform_path
    from paper_2302_02599_b200.runtime import Mesh, launch_count

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
        mesh = Mesh.from_process_group([ws])
        shape = (SHARD_ROWS_NGPU * ws, 8192)
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
        # bus bytes each rank must receive (NCCL busBW convention)
        if (a, b) == ("S0R", "RR"):
            bus = (ndev - 1) * in_bytes
        else:
            bus = (ndev - 1) * in_bytes // ndev
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
        value = step_bytes / (ms_per_step * 1e-3) / 1e9
        unit = "GB/s"
    else:
        step_bytes = sum(c["bus"] for c in convs) * ws
        value = step_bytes / (ms_per_step * 1e-3) / 1e9
        unit = "GB/s"

    # roofline of the dominant kernel (the box-copy of S0R->RR, largest share)
    dom = max(convs, key=lambda c: statistics.mean(per_conv_ms[c["name"]]))
    dom_ms = statistics.mean(per_conv_ms[dom["name"]])
    traffic = None
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists():
        entry = json.loads(tf.read_text()).get(f"n{ws}:{dom['name']}")
        traffic = entry["dram_bytes"] if entry else None
    if ws == 1:
        achieved = dom["hbm"] / (dom_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "kernel": f"{dom['kernel']} ({dom['name']}, 8 simulated devices)",
                "achieved": round(achieved, 1), "peak": hbm_peak, "peak_kind": peak_kind,
                "unit": "GB/s", "frac": round(achieved / hbm_peak, 4), "traffic": traffic,
                "algorithmic_bytes_per_launch": dom["hbm"],
                "bytes_definition": "source bytes read once + destination bytes written",
                "launch_ms": round(dom_ms, 4)}
    else:
        achieved = dom["bus"] / (dom_ms * 1e-3) / 1e9
        roof = {"bound": "nvlink", "kernel": f"{dom['name']} exchange (NCCL p2p + box_copy)",
                "achieved": round(achieved, 1), "peak": 770.0, "peak_kind": "measured peer copy (B200_PROFILING.md)",
                "unit": "GB/s", "frac": round(achieved / 770.0, 4), "traffic": traffic,
                "algorithmic_bytes_per_launch": dom["bus"], "launch_ms": round(dom_ms, 4)}

    result = {
        "metric": METRIC, "value": round(value, 1), "unit": unit, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (index-hashed bf16 bit patterns generated on device)",
        "config": {"workload": "configs[1]: mesh of 8, S0R->RR all-gather + S0R->RS0 all-to-all",
                   "tensor": list(shape), "mesh": [8] if ws == 1 else [ws],
                   "mode": "simulated 8-device mesh on 1 GPU (pack/unpack only)" if ws == 1
                   else "one process per GPU, NCCL",
                   "path": "collapsed exchange (APL_FUSE_CHAIN)",
                   "l2": "inputs 1 GiB > 126 MB L2, no flush needed" if ws == 1 else
                   "per-GPU shard 128 MiB > L2",
                   "parallelism": f"mesh[{8 if ws == 1 else ws}]"},
        "per_conversion_ms": {k: round(statistics.mean(v), 4) for k, v in per_conv_ms.items()},
        "roofline": roof,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    result["e2e"] = run_e2e(args, mesh, meta, convs, stream, ws)
    if not args.no_sweep:
        result["mesh_sweep"] = mesh_sweep(ws, rank, dev, stream, hbm_peak)
    if ws == 1:
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
        step_bytes = sum(c["bus"] for c in convs) * ws  # same metric as `value`
    else:
        step_bytes = sum(c["hbm"] for c in convs)
    return {"value": round(step_bytes / (ms * 1e-3) / 1e9, 2), "unit": "GB/s",
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
    measured 770 GB/s peer copy. Collapsed exchanges, events on the launch
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
                           frac=round(wire / ms_t / 1e6 / 770.0, 3) if wire else None)
            rows.append(row)
            conv.close()
            del ins, outs
        mesh.close()
        torch.cuda.empty_cache()
    fr = [r["frac"] for r in rows if r.get("frac") is not None]
    return {"rows": rows, "frac_min": min(fr) if fr else None,
            "frac_median": statistics.median(fr) if fr else None,
            "peak": hbm_peak if ws == 1 else 770.0,
            "kind": "pack HBM GB/s (simulated mesh)" if ws == 1 else
                    "bus GB/s per GPU (minimal one-shot bytes, NCCL)"}


# ----------------------------------------------------------------------------- CPU legs
def _cpu_sample_shape():
    # bounded sample of the same workload: 1/16 of the rows (64 MiB global)
    return (SHAPE_1GPU[0] // 16, SHAPE_1GPU[1])


def cpu_convert_once(shape, threads):
    """Reference planner path + oracle step execution in host RAM, all 8
    simulated devices; returns (seconds, algorithmic bytes)."""
    import numpy as np

    from oracle import data as O
    from oracle import ref as R

    O.set_threads(threads)
    g = O.fill_global(shape, EB)
    total_s, total_b = 0.0, 0
    for a, b in CONVERSIONS:
        ins = O.shards(g, O.parse_spec(a, 1), [8])
        t0 = time.perf_counter()
        if R.available():
            rc, steps, _ = R.find_path([8], list(shape), EB, a, b)
            assert rc == 0
        else:
            steps = [(0, 0, -1, 0, "R")] if b == "RR" else [(3, 0, 1, 0, "RS0")]
        outs = O.replay(shape, O.parse_spec(a, 1), [8], steps, ins)
        total_s += time.perf_counter() - t0
        # same accounting as the GPU arm: distinct source bytes read + output bytes written
        total_b += sum(i.nbytes for i in ins) + sum(o.nbytes for o in outs)
    return total_s, total_b


def cpu_baseline(args):
    threads = os.cpu_count() or 1
    shape = _cpu_sample_shape()
    secs, nbytes, reps = 0.0, 0, 0
    while secs < 10.0 and reps < 50:
        s, b = cpu_convert_once(shape, threads)
        secs += s
        nbytes += b
        reps += 1
    return {"value": round(nbytes / secs / 1e9, 3), "unit": "GB/s", "cores": threads,
            "kind": "port" if not _ref_available() else "reference",
            "sample": f"{reps} x (S0R->RR + S0R->RS0) on [{shape[0]},{shape[1]}] bf16, mesh [8] "
                      f"simulated in host RAM; path from the reference planner "
                      f"({'oracle/_ref' if _ref_available() else 'n/a'}), bytes moved by the C "
                      f"oracle with {threads} threads"}


def _ref_available():
    from oracle import ref as R

    return R.available()


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    shape = _cpu_sample_shape()
    for _ in range(args.warmup):
        cpu_convert_once(shape, threads)
    secs, nbytes = 0.0, 0
    for _ in range(args.steps):
        s, b = cpu_convert_once(shape, threads)
        secs += s
        nbytes += b
    value = nbytes / secs / 1e9
    planner_us = None
    if _ref_available():
        from oracle import ref as R

        planner_us = round(1e6 * R.time_paths([8], list(SHAPE_1GPU), EB, "S0R", "RS0", 2000), 3)
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * secs / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": "configs[1]: mesh of 8, S0R->RR all-gather + S0R->RS0 all-to-all",
                   "tensor": list(shape), "mesh": [8], "mode": "host RAM, all host threads",
                   "parallelism": "cpu"},
        "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", "cores": threads,
                         "kind": "reference" if _ref_available() else "port",
                         "sample": f"per step: S0R->RR + S0R->RS0 of a [{shape[0]},{shape[1]}] "
                                   "bf16 tensor on 8 simulated devices (1/16 of the GPU "
                                   "workload); reference planner (oracle/_ref) picks the path, "
                                   "the C oracle moves the bytes"},
        "reference_planner_us_per_path": planner_us,
        "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-sweep", action="store_true", help="skip the configs 3/4 mesh sweep")
    ap.add_argument("--transport", default="peer", choices=["peer", "nccl"],
                    help="N > 1: fused peer-memory pull (default) or NCCL p2p + pack/unpack")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        run_reference(args)
    elif dist_env()[0] > 1 and args.transport == "peer":
        if not run_ours_peer(args):
            run_ours(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
