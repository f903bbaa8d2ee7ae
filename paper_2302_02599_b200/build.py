"""In-tree build of the native library (libapl.so) for sm_100a.

Compiles the host C++ (autoplan drop-in API, exchange planner, runtime,
C-ABI) with g++ and the CUDA kernels with nvcc
(-gencode arch=compute_100a,code=sm_100a -lineinfo), then links one shared
library next to this file. The library links the NCCL 2.28 that torch
itself loads (site-packages/nvidia/nccl), so one process never holds two
NCCL copies. Rebuilds only what changed (mtime of sources + headers).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = ROOT / "build" / "apl"
LIB = PKG / "libapl.so"

CUDA_HOME = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
NVCC = str(CUDA_HOME / "bin" / "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_root() -> Path:
    import importlib.util

    spec = importlib.util.find_spec("nvidia")
    roots = list(spec.submodule_search_locations) if spec else []
    for r in roots:
        p = Path(r) / "nccl"
        if (p / "include" / "nccl.h").exists():
            return p
    raise RuntimeError("NCCL headers (nvidia/nccl from the torch wheel set) not found")


def _nlohmann_include() -> Path | None:
    """Directory holding nlohmann/json.hpp (the reference's JSON library;
    in this image it ships inside cudnn_frontend's third-party tree)."""
    import importlib.util

    for cand in [Path("/usr/include"), Path("/usr/local/include")]:
        if (cand / "nlohmann" / "json.hpp").exists():
            return cand
    spec = importlib.util.find_spec("torch")
    if spec and spec.origin:
        site = Path(spec.origin).parent.parent
        for cand in [site / "include" / "cudnn_frontend" / "thirdparty"]:
            if (cand / "nlohmann" / "json.hpp").exists():
                return cand
    return None


HOST_SRCS = [
    CSRC / "host" / "mesh.cpp",
    CSRC / "host" / "spec.cpp",
    CSRC / "host" / "search.cpp",
    CSRC / "host" / "strategies.cpp",
    CSRC / "runtime" / "plan.cpp",
    CSRC / "runtime" / "runtime.cpp",
    CSRC / "runtime" / "matmul.cpp",
    CSRC / "capi.cpp",
]
CUDA_SRCS = [
    CSRC / "kernels" / "box_copy.cu",
    CSRC / "kernels" / "bulk_copy.cu",
    CSRC / "kernels" / "tile_copy.cu",
    CSRC / "kernels" / "reduce.cu",
    CSRC / "kernels" / "block_ops.cu",
    CSRC / "kernels" / "peer_sync.cu",
    CSRC / "kernels" / "gemm_tcgen05.cu",
]


def _headers() -> list[Path]:
    hs = list((ROOT / "include").rglob("*.h")) + list((ROOT / "include").rglob("*.hpp"))
    hs += list(CSRC.rglob("*.hpp")) + list(CSRC.rglob("*.cuh")) + list(CSRC.rglob("*.h"))
    return hs


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.exists() and d.stat().st_mtime > t for d in deps)


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build step failed:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")


CLI = ROOT / "paper_2302_02599_b200" / "apl_convert"


def build(verbose: bool = False, force: bool = False) -> Path:
    nccl = _nccl_root()
    incs = [f"-I{ROOT / 'include'}", f"-I{CSRC}", f"-I{CUDA_HOME / 'include'}",
            f"-I{nccl / 'include'}"]
    nl = _nlohmann_include()
    if nl is not None:
        incs.append(f"-I{nl}")
    BUILD.mkdir(parents=True, exist_ok=True)
    headers = _headers()
    jobs = []
    objs = []
    for src in HOST_SRCS:
        if not src.exists():
            continue
        obj = BUILD / (src.stem + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + headers):
            jobs.append(["g++", "-std=c++20", "-O3", "-fPIC", "-Wall", "-Wextra", "-g",
                         *incs, "-c", str(src), "-o", str(obj)])
    for src in CUDA_SRCS:
        if not src.exists():
            continue
        obj = BUILD / (src.stem + ".cu.o")
        objs.append(obj)
        if force or _stale(obj, [src] + headers):
            jobs.append([NVCC, "-std=c++20", "-O3", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC",
                         "--expt-relaxed-constexpr", *incs, "-c", str(src), "-o", str(obj)])
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        for cmd, fut in [(c, ex.submit(_run, c)) for c in jobs]:
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            fut.result()
    if force or jobs or _stale(LIB, objs):
        _run([NVCC, "-shared", *ARCH, "-o", str(LIB), *map(str, objs),
              f"-L{nccl / 'lib'}", "-l:libnccl.so.2",
              "-Xlinker", f"-rpath,{nccl / 'lib'}"])
    # the `plan convert` CLI with an execute mode (tools/apl_convert.cpp)
    cli_src = ROOT / "tools" / "apl_convert.cpp"
    if cli_src.exists() and (force or _stale(CLI, [cli_src, LIB] + headers)):
        _run(["g++", "-std=c++20", "-O2", f"-I{ROOT / 'include'}", f"-I{CUDA_HOME / 'include'}",
              str(cli_src), f"-L{LIB.parent}", "-lapl", f"-L{CUDA_HOME / 'lib64'}", "-lcudart",
              f"-Wl,-rpath,{LIB.parent}", f"-Wl,-rpath,{CUDA_HOME / 'lib64'}", "-o", str(CLI)])
    return LIB


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))
