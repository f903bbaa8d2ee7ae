"""Python face of the drop-in layout API (reference proj/include/autoplan/
layout.hpp:32-132, cluster.hpp:46-98, graph_ir.hpp:33-43, errors.hpp).

Every computation goes through libapl.so (the C++ autoplan implementation
behind include/apl.h); these classes are value holders with the reference's
names so tests read like the reference's own (proj/tests/test_layout.cpp).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Sequence

from . import _capi as A


# ---- errors (reference errors.hpp:25-108) --------------------------------
class PlanError(RuntimeError):
    pass


class SchemaError(PlanError):
    pass


class AxisError(PlanError):
    pass


class ShapeError(PlanError):
    pass


class RankMismatchError(PlanError):
    pass


class InfeasibleError(PlanError):
    pass


class CudaError(RuntimeError):
    pass


class NcclError(RuntimeError):
    pass


class ArgumentError(ValueError):
    pass


_ERRORS = {A.ERR_SCHEMA: SchemaError, A.ERR_AXIS: AxisError, A.ERR_SHAPE: ShapeError,
           A.ERR_RANK: RankMismatchError, A.ERR_INFEASIBLE: InfeasibleError,
           A.ERR_CUDA: CudaError, A.ERR_NCCL: NcclError, A.ERR_ARG: ArgumentError,
           A.ERR_PLAN: PlanError, A.ERR_INTERNAL: RuntimeError}


def check(rc: int) -> None:
    if rc != A.OK:
        msg = A.lib().apl_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, RuntimeError)(msg)


# ---- value types ------------------------------------------------------------
class CollectiveKind(enum.IntEnum):
    kAllGather = 0
    kAllReduce = 1
    kReduceScatter = 2
    kAllToAll = 3
    kShardSlice = 4

    def __str__(self) -> str:  # reference cluster.cpp:118-127 names
        return ["all-gather", "all-reduce", "reduce-scatter", "all-to-all",
                "shard-slice"][int(self)]


@dataclass
class TensorMeta:
    shape: tuple
    dtype_bytes: int = 4
    requires_grad: bool = False

    def rank(self) -> int:
        return len(self.shape)

    def num_elements(self) -> int:
        n = 1
        for e in self.shape:
            n *= int(e)
        return n

    def bytes(self) -> int:
        return self.num_elements() * self.dtype_bytes

    def c(self) -> A.Meta:
        if not 1 <= len(self.shape) <= A.MAX_DIMS:
            raise ArgumentError("tensor rank outside [1, 8]")
        m = A.Meta()
        m.rank = len(self.shape)
        m.dtype_bytes = self.dtype_bytes
        for i, e in enumerate(self.shape):
            m.shape[i] = int(e)
        return m


@dataclass
class DeviceMesh:
    shape: tuple
    axis_alpha: list = field(default_factory=list)
    axis_beta_inv: list = field(default_factory=list)
    device_flops_per_s: float = 1e12

    @staticmethod
    def uniform(shape: Sequence[int], alpha: float = 1e-5, beta_inv: float = 1e-9,
                device_flops_per_s: float = 1e12) -> "DeviceMesh":
        shape = tuple(int(s) for s in shape)
        return DeviceMesh(shape, [alpha] * len(shape), [beta_inv] * len(shape),
                          device_flops_per_s)

    def rank(self) -> int:
        return len(self.shape)

    def num_devices(self) -> int:
        n = 1
        for e in self.shape:
            n *= e
        return n

    def axis_extent(self, axis: int) -> int:
        if not 0 <= axis < len(self.shape):
            raise AxisError(f"mesh axis {axis} is outside a rank-{len(self.shape)} mesh")
        return self.shape[axis]

    def shape_string(self) -> str:
        return "x".join(str(s) for s in self.shape)

    def coord_of(self, device: int) -> tuple:
        out = []
        for n in reversed(self.shape):
            out.append(device % n)
            device //= n
        return tuple(reversed(out))

    def device_of(self, coord: Sequence[int]) -> int:
        d = 0
        for c, n in zip(coord, self.shape):
            d = d * n + c
        return d

    @property
    def assignment(self) -> list:
        return [f"d{i}" for i in range(self.num_devices())]

    def to_json(self) -> str:
        """Reference mesh_to_json (cluster.cpp:417-425) through the C-ABI."""
        n = C.c_size_t()
        check(A.lib().apl_mesh_to_json(C.byref(self.c()), self.device_flops_per_s, None, 0,
                                       C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        check(A.lib().apl_mesh_to_json(C.byref(self.c()), self.device_flops_per_s, buf,
                                       n.value + 1, C.byref(n)))
        return buf.value.decode()

    @staticmethod
    def from_json(text: str) -> "DeviceMesh":
        """Reference mesh_from_json (cluster.cpp:427-450): SchemaError on a
        malformed or inconsistent document."""
        m, fl = A.MeshDesc(), C.c_double()
        check(A.lib().apl_mesh_from_json(text.encode(), C.byref(m), C.byref(fl)))
        return DeviceMesh(tuple(m.shape[:m.ndim]), list(m.alpha[:m.ndim]),
                          list(m.beta_inv[:m.ndim]), fl.value)

    def c(self) -> A.MeshDesc:
        if not 1 <= len(self.shape) <= A.MAX_MESH:
            raise ArgumentError("mesh rank outside [1, 8]")
        m = A.MeshDesc()
        m.ndim = len(self.shape)
        for i, e in enumerate(self.shape):
            m.shape[i] = e
            m.alpha[i] = self.axis_alpha[i] if self.axis_alpha else 1e-5
            m.beta_inv[i] = self.axis_beta_inv[i] if self.axis_beta_inv else 1e-9
        return m


def parse_mesh_shape(text: str) -> tuple:
    buf = (C.c_int64 * A.MAX_MESH)()
    n = C.c_int()
    check(A.lib().apl_parse_mesh_shape(text.encode(), buf, A.MAX_MESH, C.byref(n)))
    return tuple(buf[i] for i in range(n.value))


@dataclass(frozen=True)
class DimSpec:
    axes: tuple = ()

    def replicated(self) -> bool:
        return not self.axes

    def to_string(self) -> str:
        return "R" if not self.axes else "S" + "".join(str(a) for a in self.axes)


@dataclass(frozen=True)
class ShardingSpec:
    dims: tuple
    mesh_rank: int

    @staticmethod
    def replicated(tensor_rank: int, mesh_rank: int) -> "ShardingSpec":
        return ShardingSpec(tuple(DimSpec() for _ in range(tensor_rank)), mesh_rank)

    @staticmethod
    def parse(text: str, mesh_rank: int) -> "ShardingSpec":
        s = A.Spec()
        check(A.lib().apl_spec_parse(text.encode(), mesh_rank, C.byref(s)))
        return ShardingSpec.from_c(s)

    @staticmethod
    def from_c(s: A.Spec) -> "ShardingSpec":
        dims = tuple(DimSpec(tuple(s.axes[d][i] for i in range(s.naxes[d])))
                     for d in range(s.rank))
        return ShardingSpec(dims, s.mesh_rank)

    def c(self) -> A.Spec:
        if not 1 <= len(self.dims) <= A.MAX_DIMS:
            raise ArgumentError("tensor rank outside [1, 8]")
        s = A.Spec()
        s.rank = len(self.dims)
        s.mesh_rank = self.mesh_rank
        for d, dim in enumerate(self.dims):
            s.naxes[d] = len(dim.axes)
            for i, a in enumerate(dim.axes):
                s.axes[d][i] = a
        return s

    def tensor_rank(self) -> int:
        return len(self.dims)

    def to_string(self) -> str:
        buf = C.create_string_buffer(8 * A.MAX_DIMS * (A.MAX_MESH + 1) + 1)
        check(A.lib().apl_spec_to_string(C.byref(self.c()), buf, len(buf)))
        return buf.value.decode()

    __str__ = to_string

    def used_axes(self) -> list:
        return sorted(a for d in self.dims for a in d.axes)

    def shard_count(self, mesh: DeviceMesh) -> int:
        n = 1
        for a in self.used_axes():
            n *= mesh.axis_extent(a)
        return n

    def per_device_bytes(self, meta: TensorMeta, mesh: DeviceMesh) -> int:
        out = C.c_int64()
        check(A.lib().apl_spec_per_device_bytes(C.byref(self.c()), C.byref(mesh.c()),
                                                C.byref(meta.c()), C.byref(out)))
        return out.value

    def valid_for(self, meta: TensorMeta, mesh: DeviceMesh) -> bool:
        if len(self.dims) != len(meta.shape) or self.mesh_rank != len(mesh.shape):
            return False
        if any(len(d.axes) > A.MAX_MESH for d in self.dims):
            return False
        out = C.c_int()
        check(A.lib().apl_spec_valid(C.byref(self.c()), C.byref(mesh.c()), C.byref(meta.c()),
                                     C.byref(out)))
        return bool(out.value)

    def local_shape(self, meta: TensorMeta, mesh: DeviceMesh) -> tuple:
        out = []
        for d, dim in enumerate(self.dims):
            split = 1
            for a in dim.axes:
                split *= mesh.shape[a]
            out.append(meta.shape[d] // split)
        return tuple(out)


@dataclass
class TransformStep:
    kind: CollectiveKind
    tensor_dim: int
    target_dim: int
    mesh_axis: int
    result: ShardingSpec

    @staticmethod
    def from_c(s: A.Step) -> "TransformStep":
        return TransformStep(CollectiveKind(s.kind), s.tensor_dim, s.target_dim, s.mesh_axis,
                             ShardingSpec.from_c(s.result))

    def c(self) -> A.Step:
        s = A.Step()
        s.kind = int(self.kind)
        s.tensor_dim = self.tensor_dim
        s.target_dim = self.target_dim
        s.mesh_axis = self.mesh_axis
        s.result = self.result.c()
        return s

    def describe(self) -> str:
        tail = f"->{self.target_dim}" if self.kind == CollectiveKind.kAllToAll else ""
        return f"{self.kind} d{self.tensor_dim}{tail} ax{self.mesh_axis} => {self.result}"


@dataclass
class TransformPath:
    source: ShardingSpec
    target: ShardingSpec
    steps: list = field(default_factory=list)
    comm_cost_s: float = 0.0

    def steps_c(self):
        arr = (A.Step * max(1, len(self.steps)))()
        for i, s in enumerate(self.steps):
            arr[i] = s.c()
        return arr


@dataclass
class DimDiffWeights:
    all_gather: float = 2
    shard: float = 1
    all_to_all: float = 2
    step_penalty: float = 2

    def c(self):
        return (C.c_double * 4)(self.all_gather, self.shard, self.all_to_all, self.step_penalty)


_STEP_CAP = 64


def one_step_transforms(spec: ShardingSpec, mesh: DeviceMesh, meta: TensorMeta) -> list:
    cap = 256
    arr = (A.Step * cap)()
    n = C.c_int()
    check(A.lib().apl_one_step_transforms(C.byref(spec.c()), C.byref(mesh.c()),
                                          C.byref(meta.c()), arr, cap, C.byref(n)))
    return [(ShardingSpec.from_c(arr[i].result), TransformStep.from_c(arr[i]))
            for i in range(n.value)]


def dim_diff(src: DimSpec, tgt: DimSpec, weights: DimDiffWeights | None = None) -> float:
    a = (C.c_int32 * max(1, len(src.axes)))(*src.axes)
    b = (C.c_int32 * max(1, len(tgt.axes)))(*tgt.axes)
    out = C.c_double()
    w = weights.c() if weights else None
    check(A.lib().apl_dim_diff(a, len(src.axes), b, len(tgt.axes), w, C.byref(out)))
    return out.value


def heuristic_diff(src: ShardingSpec, tgt: ShardingSpec,
                   weights: DimDiffWeights | None = None) -> float:
    out = C.c_double()
    w = weights.c() if weights else None
    check(A.lib().apl_heuristic_diff(C.byref(src.c()), C.byref(tgt.c()), w, C.byref(out)))
    return out.value


def _emit(src, tgt, arr, n, cost) -> TransformPath:
    return TransformPath(src, tgt, [TransformStep.from_c(arr[i]) for i in range(n.value)],
                         cost.value)


def find_transform_path(src: ShardingSpec, tgt: ShardingSpec, mesh: DeviceMesh,
                        meta: TensorMeta) -> TransformPath:
    """find_transform_path + conversion_cost (the path comes back priced)."""
    arr = (A.Step * _STEP_CAP)()
    n = C.c_int()
    cost = C.c_double()
    check(A.lib().apl_find_transform_path(C.byref(mesh.c()), C.byref(src.c()),
                                          C.byref(tgt.c()), C.byref(meta.c()), arr, _STEP_CAP,
                                          C.byref(n), C.byref(cost)))
    return _emit(src, tgt, arr, n, cost)


def collective_cost(mesh: DeviceMesh, axes: Sequence[int], kind: CollectiveKind,
                    bytes_: float) -> float:
    ax = (C.c_int32 * max(1, len(axes)))(*axes)
    out = C.c_double()
    check(A.lib().apl_collective_cost(C.byref(mesh.c()), ax, len(axes), int(kind),
                                      float(bytes_), C.byref(out)))
    return out.value


def conversion_cost(path: TransformPath, mesh: DeviceMesh, meta: TensorMeta) -> float:
    """Reference layout.cpp:318-329: each step priced on the shard it sees."""
    total = 0.0
    cur = path.source
    for s in path.steps:
        total += collective_cost(mesh, [s.mesh_axis], s.kind, cur.per_device_bytes(meta, mesh))
        cur = s.result
    path.comm_cost_s = total
    return total


class PathCache:
    def __init__(self):
        h = C.c_void_p()
        check(A.lib().apl_path_cache_create(C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            A.lib().apl_path_cache_destroy(h)
            self._h = None

    def get(self, src: ShardingSpec, tgt: ShardingSpec, mesh: DeviceMesh,
            meta: TensorMeta) -> TransformPath:
        arr = (A.Step * _STEP_CAP)()
        n = C.c_int()
        cost = C.c_double()
        check(A.lib().apl_path_cache_get(self._h, C.byref(mesh.c()), C.byref(src.c()),
                                         C.byref(tgt.c()), C.byref(meta.c()), arr, _STEP_CAP,
                                         C.byref(n), C.byref(cost)))
        return _emit(src, tgt, arr, n, cost)

    def _stats(self):
        s, z = C.c_size_t(), C.c_size_t()
        check(A.lib().apl_path_cache_stats(self._h, C.byref(s), C.byref(z)))
        return s.value, z.value

    def searches(self) -> int:
        return self._stats()[0]

    def size(self) -> int:
        return self._stats()[1]

    def clear(self) -> None:
        check(A.lib().apl_path_cache_clear(self._h))


@dataclass
class Piece:
    sender: int
    receiver: int
    src_lo: tuple
    dst_lo: tuple
    ext: tuple


def plan_pieces(mesh: DeviceMesh, src: ShardingSpec, tgt: ShardingSpec, meta: TensorMeta,
                device: int, role: str = "recv") -> list:
    """Exchange plan of the direct src->tgt redistribution for one device."""
    cap = max(16, mesh.num_devices() * 4)
    while True:
        arr = (A.PieceC * cap)()
        n = C.c_int()
        rc = A.lib().apl_plan_pieces(C.byref(mesh.c()), C.byref(src.c()), C.byref(tgt.c()),
                                     C.byref(meta.c()), device, 0 if role == "recv" else 1,
                                     arr, cap, C.byref(n))
        if rc == A.ERR_ARG and n.value > cap:
            cap = n.value
            continue
        check(rc)
        k = len(meta.shape)
        return [Piece(arr[i].sender, arr[i].receiver, tuple(arr[i].src_lo[:k]),
                      tuple(arr[i].dst_lo[:k]), tuple(arr[i].ext[:k])) for i in range(n.value)]


def conversion_schedule(mesh: DeviceMesh, rank: int, path: "TransformPath", meta: TensorMeta,
                        fuse: bool) -> dict:
    """Dry run of the distributed executor for `rank`: every hop of the
    conversion (collapsed exchange, point-to-point step exchanges, or
    all-gathers on an axis communicator) with its copies and transfers."""
    import json

    n = C.c_size_t()
    cap = 1 << 16
    steps = path.steps_c()
    while True:
        buf = C.create_string_buffer(cap)
        rc = A.lib().apl_conversion_schedule_json(
            C.byref(mesh.c()), rank, C.byref(path.source.c()), C.byref(path.target.c()), steps,
            len(path.steps), C.byref(meta.c()), A.FUSE_CHAIN if fuse else A.STEPWISE, buf, cap,
            C.byref(n))
        if rc == A.ERR_ARG and n.value > cap:
            cap = n.value
            continue
        check(rc)
        return json.loads(buf.value.decode())


def exchange_schedule(mesh: DeviceMesh, rank: int, src: ShardingSpec, tgt: ShardingSpec,
                      meta: TensorMeta) -> dict:
    """Dry run of the distributed executor's schedule for `rank` (host only)."""
    import json

    n = C.c_size_t()
    cap = 1 << 16
    while True:
        buf = C.create_string_buffer(cap)
        rc = A.lib().apl_exchange_schedule_json(C.byref(mesh.c()), rank, C.byref(src.c()),
                                                C.byref(tgt.c()), C.byref(meta.c()), buf, cap,
                                                C.byref(n))
        if rc == A.ERR_ARG and n.value > cap:
            cap = n.value
            continue
        check(rc)
        return json.loads(buf.value.decode())
