"""Sharded-matmul strategies (reference OpStrategy, intraop.hpp:34-49) and the
catalog (intraop.cpp:141-234, 497-555), computed by libapl.so. Torch-free."""
from __future__ import annotations

import ctypes as C
from typing import Sequence

from . import _capi as A
from .layout import DeviceMesh, ShardingSpec, TensorMeta, check


class MatmulStrategy:
    """A reference-catalog strategy (OpStrategy, intraop.hpp:34-49) with specs
    on the logical A[..m.., k], B[k, n], C[..m.., n]."""

    def __init__(self, name: str, a: ShardingSpec, b: ShardingSpec, c: ShardingSpec,
                 reduce_axes: Sequence[int] = ()):
        self.name, self.a, self.b, self.c = name, a, b, c
        self.reduce_axes = tuple(reduce_axes)

    @property
    def partial_sum(self) -> bool:
        return bool(self.reduce_axes)

    def c_struct(self) -> A.MatmulStrategyC:
        s = A.MatmulStrategyC()
        s.a, s.b, s.c = self.a.c(), self.b.c(), self.c.c()
        s.partial_sum = 1 if self.reduce_axes else 0
        s.nreduce = len(self.reduce_axes)
        for i, ax in enumerate(self.reduce_axes):
            s.reduce_axes[i] = ax
        return s

    def __repr__(self) -> str:
        return (f"MatmulStrategy({self.name}: {self.a} x {self.b} -> {self.c}"
                f"{' partial over ' + str(self.reduce_axes) if self.reduce_axes else ''})")



    # catalog pricing (filled by matmul_strategies)
    compute_time_s: float = 0.0
    comm_time_s: float = 0.0
    memory_bytes: int = 0


def matmul_strategies(mesh: DeviceMesh, a: TensorMeta, b: TensorMeta, batched: bool = False,
                      device_flops_per_s: float | None = None) -> list:
    """Every valid strategy in the reference catalog's order."""
    cap = 4096
    arr = (A.StrategyInfoC * cap)()
    n = C.c_int()
    rate = mesh.device_flops_per_s if device_flops_per_s is None else device_flops_per_s
    check(A.lib().apl_matmul_strategies(C.byref(mesh.c()), C.byref(a.c()), C.byref(b.c()),
                                        1 if batched else 0, rate, arr, cap, C.byref(n)))
    out = []
    for i in range(n.value):
        info = arr[i]
        st = info.strategy
        red = [st.reduce_axes[j] for j in range(st.nreduce)]
        m = MatmulStrategy(info.name.decode(), ShardingSpec.from_c(st.a), ShardingSpec.from_c(st.b),
                           ShardingSpec.from_c(st.c), red)
        m.compute_time_s = info.compute_time_s
        m.comm_time_s = info.comm_time_s
        m.memory_bytes = info.memory_bytes
        out.append(m)
    return out


def find_matmul_strategy(name: str, mesh: DeviceMesh, a: TensorMeta, b: TensorMeta,
                         batched: bool = False) -> MatmulStrategy:
    for s in matmul_strategies(mesh, a, b, batched):
        if s.name == name:
            return s
    raise KeyError(f"no valid matmul strategy named {name!r} for these shapes")
