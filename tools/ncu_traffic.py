"""DRAM traffic of the bench's dominant launches from one `ncu --set full`
capture, stamped with the copy-kernel source hash bench.py checks
(bench.kernel_sources_sha), so `roofline.traffic` is only reported for the
kernels that were actually profiled.

Runs on the GPU box:

    python tools/ncu_traffic.py [--out gpurun_out/traffic.json]

It profiles `bench.py --steps 1 --warmup 3 --no-sweep --no-cpu` (the N=1
workload: S0R->RR then S0R->RS0 of the [65536, 8192] bf16 tensor on a
simulated mesh of 8), keeps the last launch of each conversion's kernel and
writes {"n1:S0R->RR": {"dram_bytes", "kernel", "gpu_time_ns", "source",
"kernel_sources_sha"}, ...}. Copy the file to profiles/traffic.json to stamp
later bench runs of the same sources.
"""
import argparse
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

METRICS = ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "traffic.json"))
    args = ap.parse_args()
    import bench  # noqa: E402  (for the source stamp only; nothing runs)

    cmd = ["ncu", "--set", "full", "--clock-control", "none", "--csv", "--page", "raw",
           "--print-units", "base", "-k", "regex:box_copy|bulk_copy|tile_copy",
           sys.executable, str(ROOT / "bench.py"), "--steps", "1", "--warmup", "3",
           "--no-sweep", "--no-cpu"]
    r = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith('"')]
    if not lines:
        sys.exit(f"ncu produced no CSV rows (rc={r.returncode}):\n{r.stderr[-2000:]}")
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    head = rows[0]
    launches = []
    for row in rows[1:]:
        d = dict(zip(head, row))
        if d.get("ID", "").isdigit():
            launches.append(d)
    # each step converts S0R->RR (the all-gather fan-out: box_copy) then
    # S0R->RS0 (the all-to-all: bulk_copy); the last launch of each is warm
    out = {}
    for conv, pat in (("S0R->RR", "box_copy"), ("S0R->RS0", "bulk_copy")):
        hits = [d for d in launches if pat in d["Kernel Name"]]
        if not hits:
            continue
        d = hits[-1]
        out[f"n1:{conv}"] = {
            "dram_bytes": int(float(d["dram__bytes_read.sum"]) + float(d["dram__bytes_write.sum"])),
            "dram_read": int(float(d["dram__bytes_read.sum"])),
            "dram_write": int(float(d["dram__bytes_write.sum"])),
            "gpu_time_ns": float(d["gpu__time_duration.sum"]),
            "kernel": d["Kernel Name"][:120],
            "source": "tools/ncu_traffic.py (ncu --set full, bench.py N=1)",
            "kernel_sources_sha": bench.kernel_sources_sha(),
        }
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out))


if __name__ == "__main__":
    main()
