"""Distributed plan execution over peer memory (one process per GPU, no NCCL).

`PeerRuntime` gives `executor.PlanExecutor` the mesh interface it uses
(prepare / sharded_matmul / sharded_matmul_backward / all_reduce / empty) on
top of a `runtime.PeerMesh`:

  * a symmetric heap: one IPC-exported arena per rank, mapped by every peer,
    with a deterministic bump allocator -- every rank allocates the same
    shapes in the same order (SPMD layouts have equal local shapes), so a
    tensor lives at the same offset on every rank and its peers' copies are
    `peer_base[q] + offset`;
  * conversions (the reference's insert_comm_nodes chains, planner.cpp:
    284-347) collapse to ONE launch per rank (apl_run_pull_sync): it
    announces this rank's ready flag, acquires the flags of the ranks it
    reads from, pulls the target pieces straight out of the peers' heap
    tensors and announces done from its last CTA;
  * partial sums (`<host>.ar`, planner.cpp:263-282, over any mesh-axis group)
    are ONE in-place peer all-reduce kernel per rank (apl_peer_allreduce);
  * ordering is device-side epoch flags (apl_peer_flags_*), no host barrier:
    ready before a collective reads peers, done after; the heap is recycled
    at the next forward only once every peer signalled done.
"""
from __future__ import annotations

import ctypes as C
from typing import Sequence

import torch

from . import _capi as A
from .layout import DeviceMesh, ShardingSpec, TensorMeta, check
from .runtime import PeerMesh, Mesh, MatmulStrategy, _DTYPE_CODE, _stream_handle


def _group(geo: DeviceMesh, rank: int, axes: Sequence[int]) -> list:
    """Devices differing from `rank` only on `axes`, in mixed-radix order
    (ascending device index: coordinates are row-major)."""
    me = geo.coord_of(rank)
    out = []
    for d in range(geo.num_devices()):
        c = geo.coord_of(d)
        if all(c[a] == me[a] for a in range(geo.rank()) if a not in axes):
            out.append(d)
    return out


class PeerConversion:
    """A src -> tgt conversion on the peer runtime: one pull kernel."""

    def __init__(self, rt: "PeerRuntime", src: ShardingSpec, tgt: ShardingSpec,
                 meta: TensorMeta):
        self.rt, self.src, self.tgt, self.meta = rt, src, tgt, meta

    def __call__(self, inputs, outputs, stream=None) -> None:
        self.rt.pull(self.src, self.tgt, self.meta, inputs[0], outputs[0], stream)

    def close(self) -> None:
        pass


class PeerRuntime:
    """Mesh interface of the plan executor over peer memory (see module doc)."""

    def __init__(self, shape: Sequence[int], rank: int, device: int,
                 heap_bytes: int = 4 << 30, group=None):
        self.pm = PeerMesh(shape, rank, device, 16, group=group)
        self.geo = self.pm.geo
        self.rank, self.device = rank, device
        self.num_devices = self.geo.num_devices()
        self.num_local, self.first_local, self.distributed = 1, rank, True
        self.heap, self.peer_base = self.pm.shared_buffer(heap_bytes)
        self.heap_base = self.heap.data_ptr()
        self.heap_bytes = heap_bytes
        self._off = 0
        self._local = Mesh.local([1], device=device)  # per-rank GEMMs on the local shards
        import os

        # conversions as one fused launch (APL_PEER_FUSED=0: flag kernels + pull)
        self.fused = os.environ.get("APL_PEER_FUSED", "1") != "0"

    # ---- symmetric heap ------------------------------------------------------
    def empty(self, shape, dtype) -> torch.Tensor:
        n = 1
        for e in shape:
            n *= int(e)
        nbytes = n * torch.empty((), dtype=dtype).element_size()
        off = self._off
        if off + nbytes > self.heap_bytes:
            raise MemoryError("symmetric heap exhausted (raise heap_bytes)")
        self._off = (off + nbytes + 255) // 256 * 256
        return self.heap[off:off + nbytes].view(dtype).view(*[int(e) for e in shape])

    def begin_step(self, stream=None) -> None:
        """Recycle the heap: stream-ordered wait until every peer finished
        reading this rank's heap (done flags of the last collective)."""
        if self.pm.epoch:
            self._wait(self._all_others(), self.pm.epoch, done=True, stream=stream)
        self._off = 0

    def _in_heap(self, t: torch.Tensor) -> bool:
        p = t.data_ptr()
        return self.heap_base <= p < self.heap_base + self.heap_bytes and t.is_contiguous()

    def _peer_ptrs(self, t: torch.Tensor, ranks) -> list:
        off = t.data_ptr() - self.heap_base
        return [self.peer_base[q] + off for q in ranks]

    # ---- flags -----------------------------------------------------------------
    def _all_others(self):
        return [q for q in range(self.num_devices) if q != self.rank]

    def _store(self, done: bool, stream) -> None:
        pm = self.pm
        slot = (self.num_devices if done else 0) + self.rank
        check(A.lib().apl_peer_flags_store(pm._peer_flags, pm._n_others, slot, pm.epoch,
                                           _stream_handle(stream)))

    def _wait(self, ranks, epoch, done: bool, stream) -> None:
        ranks = [q for q in ranks if q != self.rank]
        if not ranks:
            return
        base = self.num_devices if done else 0
        slots = (C.c_int32 * len(ranks))(*[base + q for q in ranks])
        check(A.lib().apl_peer_flags_wait(C.c_void_p(self.pm.flags.data_ptr()), slots, len(ranks),
                                          epoch, self.pm.timeout_ms, _stream_handle(stream)))

    # ---- conversions -----------------------------------------------------------
    def prepare(self, path, meta: TensorMeta, fuse: bool = True) -> PeerConversion:
        # the bytes of every device depend only on (tensor, target, mesh):
        # the chain always collapses to one pull on this transport
        return PeerConversion(self, path.source, path.target, meta)

    def pull(self, src, tgt, meta, x: torch.Tensor, out: torch.Tensor, stream=None) -> None:
        if not self._in_heap(x):  # e.g. a placeholder shard: stage it in the heap once
            y = self.empty(x.shape, x.dtype)
            y.copy_(x)
            x = y
        pm = self.pm
        pm.epoch += 1
        e = pm.epoch
        table = (C.c_void_p * self.num_devices)(*self._peer_ptrs(x, range(self.num_devices)))
        if self.fused:
            # one launch: announce, acquire the actual senders, pull, announce done
            sync = A.PeerSyncC(pm._all_flags, pm.flags.data_ptr(), pm._counter.data_ptr(), e,
                               pm.timeout_ms)
            check(A.lib().apl_run_pull_sync(pm._h, C.byref(src.c()), C.byref(tgt.c()),
                                            C.byref(meta.c()), table, C.c_void_p(out.data_ptr()),
                                            C.byref(sync), _stream_handle(stream)))
            return
        self._store(False, stream)
        self._wait(self._all_others(), e, False, stream)
        check(A.lib().apl_run_pull(pm._h, C.byref(src.c()), C.byref(tgt.c()), C.byref(meta.c()),
                                   table, C.c_void_p(out.data_ptr()), _stream_handle(stream)))
        self._store(True, stream)

    # ---- fused all-gather -> GEMM -------------------------------------------
    def peer_ptr(self, t: torch.Tensor, rank: int) -> int:
        """Device address of heap tensor `t` on `rank`, mapped here."""
        return self.peer_base[rank] + (t.data_ptr() - self.heap_base)

    def gather_begin(self, x: torch.Tensor, stream=None) -> torch.Tensor:
        """Publish this rank's block of a sharded operand for peers to read in
        place (staged in the heap if needed; ready flags): the all-gather of
        an all-gather -> GEMM fusion, whose GEMM then reads the owners'
        blocks over peer memory. Pair with gather_end()."""
        if not self._in_heap(x):
            y = self.empty(x.shape, x.dtype)
            y.copy_(x)
            x = y
        self.pm.epoch += 1
        self._store(False, stream)
        self._wait(self._all_others(), self.pm.epoch, False, stream)
        return x

    def gather_end(self, stream=None) -> None:
        """This rank's readers of peer blocks are done (after the GEMM)."""
        self._store(True, stream)

    # ---- partial sums ----------------------------------------------------------
    def all_reduce(self, axes: Sequence[int], tensors, stream=None) -> None:
        """In-place sum over the mesh-axis group of `axes` (one kernel)."""
        t = tensors[0]
        if not self._in_heap(t):
            raise ValueError("peer all-reduce buffers must live in the symmetric heap")
        members = _group(self.geo, self.rank, list(axes))
        P = len(members)
        pm = self.pm
        pm.epoch += 1
        e = pm.epoch
        self._store(False, stream)
        self._wait(members, e, False, stream)
        if P > 1:
            n = t.numel()
            idx = members.index(self.rank)
            per = (n // P) // 8 * 8
            lo = idx * per
            cnt = per if idx < P - 1 else n - lo
            eb = t.element_size()
            ptrs = (C.c_void_p * P)(*[p + lo * eb for p in self._peer_ptrs(t, members)])
            check(A.lib().apl_peer_allreduce(ptrs, P, cnt, _DTYPE_CODE[t.dtype],
                                             _stream_handle(stream)))
        self._store(True, stream)
        self._wait(members, e, True, stream)

    # ---- sharded matmul --------------------------------------------------------
    @staticmethod
    def _local_strategy():
        r = ShardingSpec.parse("RR", 1)
        return MatmulStrategy("local", r, r, r)

    def sharded_matmul(self, strategy: MatmulStrategy, a_meta, b_meta, a_shards, b_shards,
                       c_shards, gelu: bool = False, b_layout: str = "nk", stream=None,
                       gelu_save=None) -> None:
        a, b, c = a_shards[0], b_shards[0], c_shards[0]
        am = TensorMeta((a.numel() // a.shape[-1], a.shape[-1]), 2)
        bm = TensorMeta(tuple(b.shape) if b_layout == "kn" else (b.shape[1], b.shape[0]), 2)
        st = self._local_strategy()
        av, cv = a.reshape(am.shape), c.view(am.shape[0], -1)
        if not strategy.partial_sum:
            self._local.sharded_matmul(st, am, bm, [av], [b], [cv], gelu=gelu, b_layout=b_layout,
                                       stream=stream,
                                       gelu_save=None if gelu_save is None else
                                       [gelu_save[0].view(cv.shape)])
            return
        P = self.num_devices
        M, N = cv.shape
        if (sorted(strategy.reduce_axes) == list(range(self.geo.rank())) and 1 < P <= 8
                and M % (P * 128) == 0 and self._in_heap(c)):
            self._gemm_allreduce(av, b, cv, b_layout, stream)
        else:
            self._local.sharded_matmul(st, am, bm, [av], [b], [cv], b_layout=b_layout,
                                       stream=stream)
            self.all_reduce(strategy.reduce_axes, [c], stream=stream)
        if gelu_save is not None:
            gelu_save[0].copy_(c)
        if gelu or gelu_save is not None:
            from .runtime import gelu as gelu_fn
            gelu_fn(c, c, stream=stream)

    def _gemm_allreduce(self, a, b, c, b_layout, stream) -> None:
        """Partial sum over every rank, fused: the GEMM epilogue stores each
        fp32 row block of the partial into its owner's heap staging slab
        (reduce-scatter traffic overlapping the MMAs); each owner sums its
        slabs and stores its rows into every rank's `c` (heap, same offset)."""
        P, r = self.num_devices, self.rank
        M, N = c.shape
        rpo = M // P
        staging = self.empty((P, rpo, N), torch.float32)
        slabs = (C.c_void_p * P)(*[p + r * rpo * N * 4 for p in self._peer_ptrs(staging, range(P))])
        eb = c.element_size()
        outs = (C.c_void_p * P)(*[p + r * rpo * N * eb for p in self._peer_ptrs(c, range(P))])
        pm, lib, sh = self.pm, A.lib(), _stream_handle(stream)
        check(lib.apl_peer_gemm_scatter(C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()), slabs,
                                        P, M, N, a.shape[1], a.stride(0), b.stride(0),
                                        A.B_KN if b_layout == "kn" else A.B_NK, sh))
        pm.epoch += 1
        e = pm.epoch
        self._store(False, stream)
        self._wait(self._all_others(), e, False, stream)
        check(lib.apl_peer_reduce_gather(C.c_void_p(staging.data_ptr()), P, rpo * N, outs, P,
                                         _DTYPE_CODE[c.dtype], sh))
        self._store(True, stream)
        self._wait(self._all_others(), e, True, stream)

    def sharded_matmul_backward(self, strategy: MatmulStrategy, a_meta, b_meta, a_shards,
                                b_shards, dc_shards, da_shards=None, db_shards=None,
                                b_layout: str = "nk", gelu_aux=None, stream=None) -> None:
        a, b, dc = a_shards[0], b_shards[0], dc_shards[0]
        am = TensorMeta((a.numel() // a.shape[-1], a.shape[-1]), 2)
        bm = TensorMeta(tuple(b.shape) if b_layout == "kn" else (b.shape[1], b.shape[0]), 2)
        st = self._local_strategy()
        dcv = dc.reshape(am.shape[0], -1)
        self._local.sharded_matmul_backward(
            st, am, bm, [a.reshape(am.shape)], [b], [dcv],
            None if da_shards is None else [da_shards[0].view(am.shape)],
            None if db_shards is None else [db_shards[0]], b_layout=b_layout,
            gelu_aux=None if gelu_aux is None else [gelu_aux[0].view(am.shape)], stream=stream)
        batched = len(b_meta.shape) == 3
        n_axes = sorted(strategy.c.dims[-1].axes)
        m_axes = sorted(a for d in strategy.c.dims[(1 if batched else 0):-1] for a in d.axes)
        if da_shards is not None and n_axes:
            self.all_reduce(n_axes, da_shards, stream=stream)
        if db_shards is not None and m_axes:
            self.all_reduce(m_axes, db_shards, stream=stream)

    def close(self) -> None:
        self._local.close()
        self.pm.close()
