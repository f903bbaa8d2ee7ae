"""ctypes access to the C data oracle (oracle/_build/libapl_oracle.so).

Test infrastructure only: builds the expected bytes of every simulated
device for a conversion, two independent ways (direct slicing of the global
tensor by the target spec; step-by-step replay of the reference path).
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

LIB = Path(__file__).resolve().parent / "_build" / "libapl_oracle.so"
SEED = 2302
MAX_DIMS, MAX_MESH = 8, 8
_lib = None


class OrSpec(C.Structure):
    _fields_ = [("rank", C.c_int32), ("mesh_rank", C.c_int32),
                ("naxes", C.c_int32 * MAX_DIMS), ("axes", (C.c_int32 * MAX_MESH) * MAX_DIMS)]


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB.exists():
            import oracle

            oracle.build(ref=False)
        h = C.CDLL(str(LIB))
        I64P = C.POINTER(C.c_int64)
        h.oracle_fill.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_uint64]
        h.oracle_local.argtypes = [C.c_void_p, I64P, C.c_int, C.c_int, I64P, C.c_int,
                                   C.POINTER(OrSpec), C.c_int64, C.c_void_p]
        h.oracle_apply_step.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, I64P, C.c_int,
                                        C.c_int, I64P, C.c_int, C.POINTER(OrSpec),
                                        C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]
        h.oracle_group_sum.argtypes = [C.POINTER(C.c_void_p), C.c_int, C.c_int64, C.c_int,
                                       C.c_void_p]
        h.oracle_set_threads.argtypes = [C.c_int]
        h.oracle_num_threads.restype = C.c_int
        _lib = h
    return _lib


def parse_spec(text: str, mesh_rank: int) -> list:
    """'S01R' -> [[0, 1], []] (plain-Python restatement of the text form)."""
    dims, i = [], 0
    while i < len(text):
        if text[i] == "R":
            dims.append([])
            i += 1
        else:
            assert text[i] == "S"
            i += 1
            axes = []
            while i < len(text) and text[i].isdigit():
                axes.append(int(text[i]))
                i += 1
            dims.append(axes)
    return dims


def or_spec(dims: list, mesh_rank: int) -> OrSpec:
    s = OrSpec()
    s.rank = len(dims)
    s.mesh_rank = mesh_rank
    for d, axes in enumerate(dims):
        s.naxes[d] = len(axes)
        for i, a in enumerate(axes):
            s.axes[d][i] = a
    return s


def np_dtype(eb: int):
    return {1: np.uint8, 2: np.uint16, 4: np.uint32, 8: np.uint64}[eb]


def fill_global(shape, eb: int, seed: int = SEED) -> np.ndarray:
    n = int(np.prod(shape))
    out = np.empty(n, dtype=np_dtype(eb))
    lib().oracle_fill(out.ctypes.data, n, eb, seed)
    return out.reshape(shape)


def local_shape(shape, dims, mesh):
    out = []
    for d, axes in enumerate(dims):
        split = 1
        for a in axes:
            split *= mesh[a]
        out.append(shape[d] // split)
    return tuple(out)


def local(global_: np.ndarray, dims: list, mesh, device: int) -> np.ndarray:
    shape = global_.shape
    eb = global_.itemsize
    out = np.empty(local_shape(shape, dims, mesh), dtype=global_.dtype)
    g = np.ascontiguousarray(global_)
    lib().oracle_local(g.ctypes.data, (C.c_int64 * len(shape))(*shape), len(shape), eb,
                       (C.c_int64 * len(mesh))(*mesh), len(mesh),
                       C.byref(or_spec(dims, len(mesh))), device, out.ctypes.data)
    return out


def shards(global_: np.ndarray, dims: list, mesh) -> list:
    n = int(np.prod(mesh))
    return [local(global_, dims, mesh, d) for d in range(n)]


def apply_step(kind, tdim, target, axis, shape, dims, mesh, inputs: list, outs=None) -> list:
    """One reference step on simulated devices (C restatement). `outs`:
    optional preallocated output shards (reused across calls by the CPU
    baseline, so it times the byte movement, not page faults)."""
    new = [list(a) for a in dims]
    if kind == 0:
        new[tdim].pop()
    elif kind == 4:
        new[tdim].append(axis)
    elif kind == 3:
        new[tdim].pop()
        new[target].append(axis)
    if outs is None:
        outs = [np.empty(local_shape(shape, new, mesh), dtype=inputs[0].dtype) for _ in inputs]
    ins = (C.c_void_p * len(inputs))(*[a.ctypes.data for a in inputs])
    ops = (C.c_void_p * len(outs))(*[a.ctypes.data for a in outs])
    rc = lib().oracle_apply_step(kind, tdim, target, axis, (C.c_int64 * len(shape))(*shape),
                                 len(shape), inputs[0].itemsize, (C.c_int64 * len(mesh))(*mesh),
                                 len(mesh), C.byref(or_spec(dims, len(mesh))), ins, ops)
    assert rc == 0
    return outs, new


def replay(shape, src_dims, mesh, steps, inputs: list, outs=None) -> list:
    """Replay steps [(kind, tdim, target, axis, ...)] from src shards
    (`outs`: optional preallocated shards for the last step's result)."""
    cur, dims = inputs, [list(a) for a in src_dims]
    for i, s in enumerate(steps):
        last = outs if i + 1 == len(steps) else None
        cur, dims = apply_step(s[0], s[1], s[2], s[3], shape, dims, mesh, cur, last)
    return cur


def set_threads(n: int) -> None:
    lib().oracle_set_threads(n)


def group_sum(parts: list, dtype_code: int) -> np.ndarray:
    out = np.empty_like(parts[0])
    arr = (C.c_void_p * len(parts))(*[p.ctypes.data for p in parts])
    lib().oracle_group_sum(arr, len(parts), parts[0].size, dtype_code, out.ctypes.data)
    return out
