"""ctypes access to the REFERENCE autoplan library (oracle/_ref, test infra).

Spec-level oracle: the paths, costs, one-step sets and spec enumerations
produced by the reference's own code (proj/src/layout.cpp, cluster.cpp,
tests/helpers.hpp) compiled here from /root/reference.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

LIB = Path(__file__).resolve().parent / "_ref" / "libautoplan_ref.so"
_lib = None


def available() -> bool:
    return LIB.exists()


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        h = C.CDLL(str(LIB))
        I64P = C.POINTER(C.c_int64)
        h.ref_find_path.argtypes = [I64P, C.c_int, I64P, C.c_int, C.c_int, C.c_char_p,
                                    C.c_char_p, C.c_char_p, C.c_size_t]
        h.ref_one_step.argtypes = [I64P, C.c_int, I64P, C.c_int, C.c_int, C.c_char_p,
                                   C.c_char_p, C.c_size_t]
        h.ref_all_valid_specs.argtypes = [I64P, C.c_int, I64P, C.c_int, C.c_int, C.c_char_p,
                                          C.c_size_t]
        h.ref_bfs_min_steps.argtypes = [I64P, C.c_int, I64P, C.c_int, C.c_int, C.c_char_p,
                                        C.c_char_p]
        h.ref_dim_diff.argtypes = [C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_int), C.c_int,
                                   C.POINTER(C.c_double)]
        h.ref_heuristic_diff.argtypes = [C.c_int, C.c_char_p, C.c_char_p, C.POINTER(C.c_double)]
        h.ref_collective_cost.argtypes = [I64P, C.c_int, C.POINTER(C.c_int), C.c_int, C.c_int,
                                          C.c_double, C.POINTER(C.c_double)]
        h.ref_spec_valid.argtypes = [I64P, C.c_int, I64P, C.c_int, C.c_int, C.c_char_p]
        h.ref_time_paths.argtypes = [I64P, C.c_int, I64P, C.c_int, C.c_int, C.c_char_p,
                                     C.c_char_p, C.c_int, C.c_int]
        h.ref_time_paths.restype = C.c_double
        h.ref_mesh_json.argtypes = [C.c_char_p, C.c_char_p, C.c_size_t]
        _lib = h
    return _lib


def _arr(v):
    return (C.c_int64 * len(v))(*v)


def find_path(mesh, shape, eb, src: str, tgt: str):
    """-> (code, steps, cost); steps = [(kind, tdim, target, axis, result_text)]."""
    buf = C.create_string_buffer(1 << 16)
    rc = lib().ref_find_path(_arr(mesh), len(mesh), _arr(shape), len(shape), eb, src.encode(),
                             tgt.encode(), buf, len(buf))
    text = buf.value.decode()
    if rc != 0:
        return rc, text, None
    steps, cost = [], None
    for line in text.splitlines():
        parts = line.split()
        if parts[0] == "cost":
            cost = float(parts[1])
        else:
            steps.append((int(parts[0]), int(parts[1]), int(parts[2]), int(parts[3]), parts[4]))
    return 0, steps, cost


def one_step(mesh, shape, eb, spec: str):
    buf = C.create_string_buffer(1 << 16)
    rc = lib().ref_one_step(_arr(mesh), len(mesh), _arr(shape), len(shape), eb, spec.encode(),
                            buf, len(buf))
    if rc != 0:
        return rc, buf.value.decode()
    out = []
    for line in buf.value.decode().splitlines():
        k, d, t, a, r = line.split()
        out.append((int(k), int(d), int(t), int(a), r))
    return 0, out


def all_valid_specs(mesh, shape, eb=4):
    buf = C.create_string_buffer(1 << 20)
    rc = lib().ref_all_valid_specs(_arr(mesh), len(mesh), _arr(shape), len(shape), eb, buf,
                                   len(buf))
    assert rc == 0, buf.value
    return buf.value.decode().split()


def bfs_min_steps(mesh, shape, eb, src, tgt):
    return lib().ref_bfs_min_steps(_arr(mesh), len(mesh), _arr(shape), len(shape), eb,
                                   src.encode(), tgt.encode())


def dim_diff(a, b):
    out = C.c_double()
    lib().ref_dim_diff((C.c_int * max(1, len(a)))(*a), len(a), (C.c_int * max(1, len(b)))(*b),
                       len(b), C.byref(out))
    return out.value


def heuristic_diff(mesh_rank, a, b):
    out = C.c_double()
    rc = lib().ref_heuristic_diff(mesh_rank, a.encode(), b.encode(), C.byref(out))
    return rc, out.value


def collective_cost(mesh, axes, kind, nbytes):
    out = C.c_double()
    rc = lib().ref_collective_cost(_arr(mesh), len(mesh), (C.c_int * max(1, len(axes)))(*axes),
                                   len(axes), kind, float(nbytes), C.byref(out))
    return rc, out.value


def spec_valid(mesh, shape, eb, spec):
    return lib().ref_spec_valid(_arr(mesh), len(mesh), _arr(shape), len(shape), eb,
                                spec.encode())


def time_paths(mesh, shape, eb, src, tgt, iters=1000, hits=False) -> float:
    return lib().ref_time_paths(_arr(mesh), len(mesh), _arr(shape), len(shape), eb,
                                src.encode(), tgt.encode(), iters, 1 if hits else 0)


def mesh_json(text: str):
    """Reference mesh_from_json -> mesh_to_json: (code, canonical text or message)."""
    buf = C.create_string_buffer(1 << 16)
    rc = lib().ref_mesh_json(text.encode(), buf, len(buf))
    return rc, buf.value.decode()
