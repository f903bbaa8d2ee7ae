"""B200-native layout-conversion runtime for Colossal-Auto (arXiv 2302.02599).

Host API (drop-in names of the reference autoplan layout manager):
    DeviceMesh, TensorMeta, DimSpec, ShardingSpec, TransformStep, TransformPath,
    CollectiveKind, one_step_transforms, dim_diff, heuristic_diff,
    find_transform_path, conversion_cost, collective_cost, PathCache
Runtime (executes the paths on device data; sm_100a kernels + NCCL):
    paper_2302_02599_b200.runtime.Mesh
"""
from .layout import (AxisError, CollectiveKind, CudaError, DeviceMesh, DimDiffWeights, DimSpec,
                     InfeasibleError, NcclError, PathCache, Piece, PlanError, RankMismatchError,
                     SchemaError, ShapeError, ShardingSpec, TensorMeta, TransformPath,
                     TransformStep, collective_cost, conversion_cost, dim_diff,
                     find_transform_path, heuristic_diff, one_step_transforms,
                     parse_mesh_shape, plan_pieces)

__all__ = [n for n in dir() if not n.startswith("_")]
