"""ctypes declaration of the C-ABI in include/apl.h.

This module only loads libapl.so and declares its signatures; it never
substitutes anything for a missing library: if libapl.so is absent or was
built without sm_100a kernels the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

MAX_DIMS = 8
MAX_MESH = 8
MAX_LOCAL = 64

OK, ERR_SCHEMA, ERR_AXIS, ERR_SHAPE, ERR_RANK, ERR_INFEASIBLE, ERR_CUDA, ERR_NCCL, ERR_ARG, \
    ERR_PLAN, ERR_INTERNAL = range(11)
FUSE_CHAIN = 1
STEPWISE = 0
F32, BF16, F16 = 0, 1, 2
EPI_NONE, EPI_GELU, EPI_DGELU, EPI_GELU_SAVE = 0, 1, 2, 3
B_NK, B_KN = 0, 1


class Spec(C.Structure):
    _fields_ = [("rank", C.c_int32), ("mesh_rank", C.c_int32),
                ("naxes", C.c_int32 * MAX_DIMS), ("axes", (C.c_int32 * MAX_MESH) * MAX_DIMS)]


class Meta(C.Structure):
    _fields_ = [("rank", C.c_int32), ("dtype_bytes", C.c_int32), ("shape", C.c_int64 * MAX_DIMS)]


class Step(C.Structure):
    _fields_ = [("kind", C.c_int32), ("tensor_dim", C.c_int32), ("target_dim", C.c_int32),
                ("mesh_axis", C.c_int32), ("result", Spec)]


class MeshDesc(C.Structure):
    _fields_ = [("ndim", C.c_int32), ("shape", C.c_int64 * MAX_MESH),
                ("alpha", C.c_double * MAX_MESH), ("beta_inv", C.c_double * MAX_MESH)]


class MatmulStrategyC(C.Structure):
    _fields_ = [("a", Spec), ("b", Spec), ("c", Spec), ("partial_sum", C.c_int32),
                ("nreduce", C.c_int32), ("reduce_axes", C.c_int32 * MAX_MESH)]


class StrategyInfoC(C.Structure):
    _fields_ = [("name", C.c_char * 64), ("strategy", MatmulStrategyC),
                ("compute_time_s", C.c_double), ("comm_time_s", C.c_double),
                ("bwd_compute_time_s", C.c_double), ("bwd_comm_time_s", C.c_double),
                ("comm_buffer_bytes", C.c_int64), ("memory_bytes", C.c_int64)]


class PeerSyncC(C.Structure):
    _fields_ = [("peer_flags", C.POINTER(C.c_void_p)), ("local_flags", C.c_void_p),
                ("counter", C.c_void_p), ("epoch", C.c_uint32), ("timeout_ms", C.c_uint32)]


class PieceC(C.Structure):
    _fields_ = [("sender", C.c_int32), ("receiver", C.c_int32),
                ("src_lo", C.c_int64 * MAX_DIMS), ("dst_lo", C.c_int64 * MAX_DIMS),
                ("ext", C.c_int64 * MAX_DIMS)]


# APL_LIB: load another build (A/B timing of two builds on one box).
LIB_PATH = Path(os.environ.get("APL_LIB", Path(__file__).resolve().parent / "libapl.so"))
_lib = None

P = C.POINTER
_SIGS = {
    "apl_version": (C.c_int, []),
    "apl_last_error": (C.c_char_p, []),
    "apl_mesh_desc_uniform": (C.c_int, [P(C.c_int64), C.c_int, P(MeshDesc)]),
    "apl_parse_mesh_shape": (C.c_int, [C.c_char_p, P(C.c_int64), C.c_int, P(C.c_int)]),
    "apl_spec_parse": (C.c_int, [C.c_char_p, C.c_int, P(Spec)]),
    "apl_spec_to_string": (C.c_int, [P(Spec), C.c_char_p, C.c_size_t]),
    "apl_spec_valid": (C.c_int, [P(Spec), P(MeshDesc), P(Meta), P(C.c_int)]),
    "apl_spec_per_device_bytes": (C.c_int, [P(Spec), P(MeshDesc), P(Meta), P(C.c_int64)]),
    "apl_one_step_transforms": (C.c_int, [P(Spec), P(MeshDesc), P(Meta), P(Step), C.c_int,
                                          P(C.c_int)]),
    "apl_dim_diff": (C.c_int, [P(C.c_int32), C.c_int, P(C.c_int32), C.c_int, P(C.c_double),
                               P(C.c_double)]),
    "apl_heuristic_diff": (C.c_int, [P(Spec), P(Spec), P(C.c_double), P(C.c_double)]),
    "apl_find_transform_path": (C.c_int, [P(MeshDesc), P(Spec), P(Spec), P(Meta), P(Step),
                                          C.c_int, P(C.c_int), P(C.c_double)]),
    "apl_collective_cost": (C.c_int, [P(MeshDesc), P(C.c_int32), C.c_int, C.c_int, C.c_double,
                                      P(C.c_double)]),
    "apl_path_cache_create": (C.c_int, [P(C.c_void_p)]),
    "apl_path_cache_destroy": (C.c_int, [C.c_void_p]),
    "apl_path_cache_get": (C.c_int, [C.c_void_p, P(MeshDesc), P(Spec), P(Spec), P(Meta),
                                     P(Step), C.c_int, P(C.c_int), P(C.c_double)]),
    "apl_path_cache_stats": (C.c_int, [C.c_void_p, P(C.c_size_t), P(C.c_size_t)]),
    "apl_path_cache_clear": (C.c_int, [C.c_void_p]),
    "apl_plan_pieces": (C.c_int, [P(MeshDesc), P(Spec), P(Spec), P(Meta), C.c_int, C.c_int,
                                  P(PieceC), C.c_int, P(C.c_int)]),
    "apl_mesh_create_local": (C.c_int, [P(MeshDesc), C.c_int, P(C.c_void_p)]),
    "apl_nccl_unique_id": (C.c_int, [P(C.c_uint8)]),
    "apl_mesh_create_nccl": (C.c_int, [P(MeshDesc), C.c_int, P(C.c_uint8), C.c_int,
                                       P(C.c_void_p)]),
    "apl_mesh_to_json": (C.c_int, [P(MeshDesc), C.c_double, C.c_char_p, C.c_size_t,
                                   P(C.c_size_t)]),
    "apl_mesh_from_json": (C.c_int, [C.c_char_p, P(MeshDesc), P(C.c_double)]),
    "apl_mesh_destroy": (C.c_int, [C.c_void_p]),
    "apl_mesh_health": (C.c_int, [C.c_void_p, P(C.c_int)]),
    "apl_mesh_abort": (C.c_int, [C.c_void_p]),
    "apl_mesh_create_peer": (C.c_int, [P(MeshDesc), C.c_int, C.c_int, P(C.c_void_p)]),
    "apl_peer_alloc": (C.c_int, [C.c_void_p, C.c_size_t, P(C.c_void_p), P(C.c_uint8)]),
    "apl_peer_open": (C.c_int, [C.c_void_p, P(C.c_uint8), P(C.c_void_p)]),
    "apl_run_pull": (C.c_int, [C.c_void_p, P(Spec), P(Spec), P(Meta), P(C.c_void_p), C.c_void_p,
                               C.c_void_p]),
    "apl_run_pull_sync": (C.c_int, [C.c_void_p, P(Spec), P(Spec), P(Meta), P(C.c_void_p),
                                    C.c_void_p, P(PeerSyncC), C.c_void_p]),
    "apl_run_push_sync": (C.c_int, [C.c_void_p, P(Spec), P(Spec), P(Meta), C.c_void_p,
                                    P(C.c_void_p), P(PeerSyncC), C.c_void_p]),
    "apl_exchange_peers": (C.c_int, [C.c_void_p, P(Spec), P(Spec), P(Meta), P(C.c_int32),
                                     P(C.c_int), P(C.c_int32), P(C.c_int)]),
    "apl_mesh_info": (C.c_int, [C.c_void_p, P(C.c_int), P(C.c_int), P(C.c_int), P(C.c_int)]),
    "apl_path_workspace_bytes": (C.c_int, [C.c_void_p, P(Spec), P(Spec), P(Step), C.c_int,
                                           P(Meta), C.c_uint, P(C.c_size_t)]),
    "apl_run_step": (C.c_int, [C.c_void_p, P(Spec), P(Step), P(Meta), P(C.c_void_p),
                               P(C.c_void_p), C.c_void_p, C.c_size_t, C.c_void_p]),
    "apl_run_path": (C.c_int, [C.c_void_p, P(Spec), P(Spec), P(Step), C.c_int, P(Meta),
                               P(C.c_void_p), P(C.c_void_p), C.c_void_p, C.c_size_t, C.c_uint,
                               C.c_void_p]),
    "apl_exchange_traffic": (C.c_int, [C.c_void_p, P(Spec), P(Spec), P(Meta), P(C.c_int64),
                                       P(C.c_int64), P(C.c_int64)]),
    "apl_conversion_create": (C.c_int, [C.c_void_p, P(Spec), P(Spec), P(Step), C.c_int, P(Meta),
                                        C.c_uint, P(C.c_void_p)]),
    "apl_conversion_workspace": (C.c_int, [C.c_void_p, P(C.c_size_t)]),
    "apl_conversion_run": (C.c_int, [C.c_void_p, P(C.c_void_p), P(C.c_void_p), C.c_void_p,
                                     C.c_size_t, C.c_void_p]),
    "apl_conversion_destroy": (C.c_int, [C.c_void_p]),
    "apl_exchange_engine": (C.c_int, [C.c_void_p, P(Spec), P(Spec), P(Meta), P(C.c_int)]),
    "apl_exchange_schedule_json": (C.c_int, [P(MeshDesc), C.c_int, P(Spec), P(Spec), P(Meta),
                                             C.c_char_p, C.c_size_t, P(C.c_size_t)]),
    "apl_all_reduce": (C.c_int, [C.c_void_p, P(C.c_int32), C.c_int, P(C.c_void_p), C.c_size_t,
                                 C.c_int, C.c_void_p]),
    "apl_matmul_strategies": (C.c_int, [P(MeshDesc), P(Meta), P(Meta), C.c_int, C.c_double,
                                        P(StrategyInfoC), C.c_int, P(C.c_int)]),
    "apl_gemm_force_plan": (C.c_int, [C.c_int, C.c_int, C.c_int]),
    "apl_gemm_trace": (C.c_int, [C.c_void_p, C.c_size_t]),
    "apl_gemm_bf16": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                                C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int, C.c_int,
                                C.c_int, C.c_void_p]),
    "apl_sharded_matmul": (C.c_int, [C.c_void_p, P(MatmulStrategyC), P(Meta), P(Meta),
                                     P(C.c_void_p), P(C.c_void_p), P(C.c_void_p), C.c_int,
                                     C.c_int, C.c_int, C.c_void_p]),
    "apl_gemm_bf16_grouped": (C.c_int, [P(C.c_void_p), P(C.c_void_p), P(C.c_void_p), C.c_int,
                                        C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                        C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_int,
                                        P(C.c_void_p), C.c_void_p]),
    "apl_sharded_matmul_ex": (C.c_int, [C.c_void_p, P(MatmulStrategyC), P(Meta), P(Meta),
                                        P(C.c_void_p), P(C.c_void_p), P(C.c_void_p), C.c_int,
                                        C.c_int, C.c_int, P(C.c_void_p), C.c_void_p]),
    "apl_gelu_inplace": (C.c_int, [C.c_void_p, C.c_size_t, C.c_int, C.c_void_p]),
    "apl_gelu": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p]),
    "apl_gelu_backward": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int,
                                    C.c_void_p]),
    "apl_sharded_matmul_backward": (C.c_int, [C.c_void_p, P(MatmulStrategyC), P(Meta), P(Meta),
                                              P(C.c_void_p), P(C.c_void_p), P(C.c_void_p),
                                              P(C.c_void_p), P(C.c_void_p), C.c_int, C.c_int,
                                              P(C.c_void_p), C.c_int, C.c_void_p]),
    "apl_launch_count": (C.c_int, [P(C.c_uint64)]),
    "apl_peer_gemm_scatter": (C.c_int, [C.c_void_p, C.c_void_p, P(C.c_void_p), C.c_int,
                                        C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                        C.c_int, C.c_void_p]),
    "apl_peer_reduce_gather": (C.c_int, [C.c_void_p, C.c_int, C.c_int64, P(C.c_void_p), C.c_int,
                                         C.c_int, C.c_void_p]),
    "apl_conversion_schedule_json": (C.c_int, [P(MeshDesc), C.c_int, P(Spec), P(Spec), P(Step),
                                               C.c_int, P(Meta), C.c_uint, C.c_char_p, C.c_size_t,
                                               P(C.c_size_t)]),
    "apl_peer_allreduce": (C.c_int, [P(C.c_void_p), C.c_int, C.c_size_t, C.c_int, C.c_void_p]),
    "apl_peer_flags_store": (C.c_int, [P(C.c_void_p), C.c_int, C.c_int, C.c_uint32,
                                       C.c_void_p]),
    "apl_peer_flags_wait": (C.c_int, [C.c_void_p, P(C.c_int32), C.c_int, C.c_uint32,
                                      C.c_uint32, C.c_void_p]),
    "apl_embedding_lookup": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int64,
                                       C.c_int, C.c_void_p, C.c_void_p]),
    "apl_embedding_lookup_blocks": (C.c_int, [C.c_void_p, C.c_int64, P(C.c_void_p), C.c_int,
                                              C.c_int, C.c_int64, C.c_int64, C.c_int64,
                                              C.c_int64, C.c_int, C.c_void_p, C.c_void_p]),
    "apl_layernorm": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                C.c_int64, C.c_float, C.c_int, C.c_void_p]),
    "apl_softmax": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int,
                              C.c_void_p]),
    "apl_softmax_ex": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_float,
                                 C.c_void_p, C.c_float, C.c_int, C.c_void_p]),
    "apl_transpose": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int,
                                C.c_void_p]),
    "apl_permute": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, P(C.c_int64), P(C.c_int64),
                              C.c_int, C.c_void_p]),
    "apl_softmax_axis": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64,
                                   C.c_int, C.c_void_p]),
    "apl_softmax_axis_backward": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                            C.c_int64, C.c_int64, C.c_float, C.c_int,
                                            C.c_void_p]),
    "apl_scale": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_float, C.c_int, C.c_void_p]),
    "apl_add": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_size_t, C.c_float,
                          C.c_int, C.c_void_p]),
    "apl_layernorm_backward": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                         C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                         C.c_int64, C.c_float, C.c_int, C.c_void_p]),
    "apl_layernorm_backward_ex": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                            C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t,
                                            C.c_int64, C.c_int64, C.c_float, C.c_int,
                                            C.c_void_p]),
    "apl_layernorm_backward_scratch": (C.c_int, [C.c_int64, C.c_int64, P(C.c_size_t)]),
    "apl_softmax_backward": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                                       C.c_float, C.c_int, C.c_void_p]),
    "apl_embedding_backward": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                         C.c_int64, C.c_int64, C.c_int, C.c_void_p]),
    "apl_embedding_backward_block": (C.c_int, [P(C.c_void_p), P(C.c_void_p), C.c_int, C.c_int64,
                                               C.c_int64, C.c_void_p, C.c_int64, C.c_int64,
                                               C.c_int64, C.c_int64, C.c_int, C.c_void_p]),
    "apl_gemm_bf16_grouped_ex": (C.c_int, [P(C.c_void_p), P(C.c_void_p), P(C.c_void_p), C.c_int,
                                           C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                           C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_int,
                                           C.c_void_p]),
    "apl_mask_not": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
}

# Symbols every build must export (tests check the .so against include/apl.h).
EXPORTED = tuple(_SIGS)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build the native library first "
                "(python -c 'import __graft_entry__ as g; g.build()'); there is no fallback")
        handle = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib
