"""Per-kernel SASS instruction histogram of the built objects (evidence that
the kernels use tcgen05 / TMA / TMEM on sm_100a).

    python tools/sass_histogram.py [--out profiles/r02_sass_histogram.txt]

Runs `cuobjdump -sass` over every kernel object under build/apl/ (the nvcc
outputs that libapl.so links) and counts, per kernel, the Blackwell-specific
mnemonics: UTC*MMA (tcgen05.mma), LDTM/STTM (tcgen05.ld/st), UTMALDG/UTMASTG
(TMA tensor), UBLKCP (TMA bulk), UTMACCTL.PF (tensormap prefetch), plus the plain
LDG/STG widths and legacy HMMA (which must be absent). The header records the
source hash of each object so a stale listing is visible.
"""
from __future__ import annotations

import argparse
import collections
import hashlib
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
BUILD = ROOT / "build" / "apl"
CSRC = ROOT / "paper_2302_02599_b200" / "csrc" / "kernels"

PATTERNS = [
    ("UTC*MMA", re.compile(r"\bUTC\w*MMA\b")),
    ("UTCHMMA.2CTA", re.compile(r"\bUTC\w*MMA\.2CTA\b")),
    ("LDTM", re.compile(r"\bLDTM\b")),
    ("STTM", re.compile(r"\bSTTM\b")),
    ("UTMALDG", re.compile(r"\bUTMALDG\b")),
    ("UTMASTG", re.compile(r"\bUTMASTG\b")),
    ("UBLKCP", re.compile(r"\bUBLKCP\b")),
    ("UTMACCTL.PF", re.compile(r"\bUTMACCTL\.PF\b")),
    ("SYNCS", re.compile(r"\bSYNCS\b")),
    ("LDG.128", re.compile(r"\bLDG(?:\.[A-Z0-9_]+)*\.128\b")),
    ("STG.128", re.compile(r"\bSTG(?:\.[A-Z0-9_]+)*\.128\b")),
    ("LDG", re.compile(r"\bLDG(?:\.[A-Z0-9_]+)*(?=[\s;])")),
    ("STG", re.compile(r"\bSTG(?:\.[A-Z0-9_]+)*(?=[\s;])")),
    ("LDGSTS", re.compile(r"\bLDGSTS\b")),
    ("LDS", re.compile(r"\bLDS\b")),
    ("SHFL", re.compile(r"\bSHFL\b")),
    ("HMMA(legacy)", re.compile(r"\bHMMA\b")),
]


def demangle(names: list[str]) -> list[str]:
    try:
        out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True,
                             text=True, check=True).stdout.splitlines()
        return out if len(out) == len(names) else names
    except (OSError, subprocess.CalledProcessError):
        return names


def histogram(obj: Path) -> dict[str, collections.Counter]:
    sass = subprocess.run(["cuobjdump", "-sass", str(obj)], capture_output=True, text=True,
                          check=True).stdout
    kernels: dict[str, collections.Counter] = {}
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            kernels[cur] = collections.Counter()
            continue
        if cur is None or "/*" not in line:
            continue
        for name, pat in PATTERNS:
            if pat.search(line):
                kernels[cur][name] += 1
    return kernels


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    lines = ["# SASS instruction histogram (cuobjdump -sass, sm_100a), per kernel",
             "# columns: " + ", ".join(n for n, _ in PATTERNS), ""]
    objs = sorted(BUILD.glob("*.cu.o")) or sorted(BUILD.glob("*.o"))
    if not objs:
        print("no objects under build/apl: run __graft_entry__.build() first", file=sys.stderr)
        return 1
    for obj in objs:
        src = CSRC / obj.name.replace(".o", "")
        h = hashlib.sha256(src.read_bytes()).hexdigest()[:12] if src.exists() else "?"
        ks = histogram(obj)
        if not ks:
            continue
        lines.append(f"## {obj.name}  (source sha256 {h})")
        names = list(ks)
        for raw, pretty in zip(names, demangle(names)):
            c = ks[raw]
            cols = "  ".join(f"{n}={c[n]}" for n, _ in PATTERNS if c[n])
            lines.append(f"{pretty[:150]}\n    {cols or '(none of the tracked mnemonics)'}")
        lines.append("")
    text = "\n".join(lines)
    if args.out:
        Path(args.out).write_text(text)
    print(text)
    return 0


if __name__ == "__main__":
    sys.exit(main())
