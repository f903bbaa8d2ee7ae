"""The C-ABI boundary: libapl.so loads on CPU and exports exactly what
include/apl.h declares; argument/limit errors come back as status codes."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

from paper_2302_02599_b200 import _capi as A
from paper_2302_02599_b200 import layout as L

ROOT = Path(__file__).resolve().parent.parent


def declared_functions():
    text = (ROOT / "include" / "apl.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*|uint64_t)\s+(apl_\w+)\(", text,
                                 re.M)))


def test_header_and_binding_agree():
    assert set(declared_functions()) == set(A.EXPORTED)


def test_library_exports_every_declared_symbol():
    lib = A.lib()
    for name in declared_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", str(A.LIB_PATH)], capture_output=True,
                         text=True).stdout
    for name in declared_functions():
        assert re.search(rf"\bT {name}\b", out), name


def test_library_targets_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", str(A.LIB_PATH)], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    arches = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert arches == {"100a"}, arches


def test_status_codes_map_to_reference_error_classes():
    lib = A.lib()
    s = A.Spec()
    assert lib.apl_spec_parse(b"S9R", 2, C.byref(s)) == A.ERR_AXIS
    assert b"out of range" in lib.apl_last_error()
    assert lib.apl_spec_parse(b"XR", 2, C.byref(s)) == A.ERR_SCHEMA
    assert lib.apl_spec_parse(None, 2, C.byref(s)) == A.ERR_ARG
    mesh = L.DeviceMesh.uniform([2, 4]).c()
    meta = L.TensorMeta((4, 8), 4).c()
    src, tgt = L.ShardingSpec.parse("S0R", 2).c(), L.ShardingSpec.parse("S01R", 2).c()
    steps = (A.Step * 8)()
    n, cost = C.c_int(), C.c_double()
    assert lib.apl_find_transform_path(C.byref(mesh), C.byref(src), C.byref(tgt), C.byref(meta),
                                       steps, 8, C.byref(n), C.byref(cost)) == A.ERR_SHAPE
    # capacity too small is an argument error, with the needed count reported
    meta = L.TensorMeta((8, 8), 4).c()
    tgt = L.ShardingSpec.parse("RR", 2).c()
    assert lib.apl_find_transform_path(C.byref(mesh), C.byref(src), C.byref(tgt), C.byref(meta),
                                       steps, 0, C.byref(n), C.byref(cost)) == A.ERR_ARG
    assert n.value == 1
    bad = A.Meta()
    bad.rank, bad.dtype_bytes = 2, 3
    assert lib.apl_spec_valid(C.byref(src), C.byref(mesh), C.byref(bad), C.byref(n)) == A.ERR_ARG


def test_runtime_refuses_without_gpu_instead_of_falling_back():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib = A.lib()
    h = C.c_void_p()
    rc = lib.apl_mesh_create_local(C.byref(L.DeviceMesh.uniform([2, 2]).c()), 0, C.byref(h))
    assert rc in (A.ERR_CUDA, A.ERR_ARG)


def test_block_entry_points_validate_arguments_without_a_gpu():
    """The transformer-block entry points reject bad arguments with
    APL_ERR_ARG before touching the device (host-side validation)."""
    lib = A.lib()
    P = C.c_void_p
    one = P(16)  # never dereferenced: validation fails first
    err = A.ERR_ARG
    assert lib.apl_layernorm(one, None, None, one, 4, 8, 1e-5, 7, None) == err  # dtype
    assert lib.apl_layernorm(one, None, None, one, 4, 0, 1e-5, A.BF16, None) == err  # width
    assert lib.apl_softmax_ex(one, one, 4, 0, 1.0, None, 0.0, A.BF16, None) == err
    assert lib.apl_transpose(one, one, 1, 4, 4, 2, None) == err  # in place
    assert lib.apl_transpose(one, P(32), 1, 4, 4, 3, None) == err  # element size
    assert lib.apl_embedding_lookup(one, 4, one, 10, 8, 3, one, None) == err
    blocks = (P * 65)(*([16] * 65))
    assert lib.apl_embedding_lookup_blocks(one, 4, blocks, 65, 1, 65, 8, 0, 8, 2, one,
                                           None) == err  # > 64 blocks
    assert lib.apl_embedding_lookup_blocks(one, 4, blocks, 2, 1, 65, 8, 0, 8, 2, one,
                                           None) == err  # vocab not divisible
    assert lib.apl_embedding_lookup_blocks(one, 4, blocks, 1, 1, 64, 8, 4, 8, 2, one,
                                           None) == err  # slice outside the table
    assert lib.apl_layernorm_backward(one, None, one, one, P(16), None, None, 4, 8, 1e-5,
                                      A.BF16, None) == err  # dgamma without stats scratch
    assert lib.apl_layernorm_backward_ex(one, None, one, one, P(16), None, one, 8, 4, 8, 1e-5,
                                         A.BF16, None) == err  # stats scratch too small
    ptrs = (P * 1)(16)
    assert lib.apl_gemm_bf16_grouped_ex(ptrs, ptrs, ptrs, 1, 8, 8, 8, 4, 8, 8, 0, 1, A.BF16,
                                        None) == err  # lda < K (A as [M, K])
    assert lib.apl_gemm_bf16_grouped_ex(ptrs, ptrs, ptrs, 1, 8, 8, 8, 8, 8, 8, 5, 1, A.BF16,
                                        None) == err  # A layout
    for fn in ("apl_layernorm", "apl_softmax_ex", "apl_embedding_lookup_blocks",
               "apl_gemm_bf16_grouped_ex"):
        assert hasattr(lib, fn)
    assert lib.apl_last_error()  # a message is recorded
