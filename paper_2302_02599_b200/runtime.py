"""Torch-facing runtime over the C-ABI: meshes, conversion execution,
partial-sum all-reduce.

Device memory, streams and process groups come from torch; every byte is
moved by libapl.so kernels / NCCL calls issued from C++. There is no CPU or
eager-torch fallback: without a GPU or without libapl.so these calls raise.
"""
from __future__ import annotations

import ctypes as C
import itertools
from typing import Sequence

import torch

from . import _capi as A
from .layout import (DeviceMesh, ShardingSpec, TensorMeta, TransformPath, TransformStep,
                     check, find_transform_path)
from .strategies import MatmulStrategy  # noqa: F401  (re-exported)

_DTYPE_CODE = {torch.float32: A.F32, torch.bfloat16: A.BF16, torch.float16: A.F16}


def _ptrs(tensors: Sequence[torch.Tensor]):
    arr = (C.c_void_p * max(1, len(tensors)))()
    for i, t in enumerate(tensors):
        arr[i] = t.data_ptr()
    return arr


def _stream_handle(stream) -> C.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def gemm_grouped(a_ptrs, b_ptrs, c_ptrs, reduce: int, M: int, N: int, K: int, lda: int,
                 ldb: int, ldc: int, b_layout: str = "kn", out_dtype=torch.bfloat16,
                 gelu: bool = False, stream=None) -> None:
    """Grouped tcgen05 GEMM over raw device pointers (apl_gemm_bf16_grouped):
    C[g] = epi(sum_r A[g*reduce+r] . B[g*reduce+r]). Used for all-gather ->
    GEMM fusion: B[r] are the owner buffers of a sharded weight's K-slices."""
    P = C.c_void_p
    arr = lambda xs: (P * len(xs))(*xs)  # noqa: E731
    check(A.lib().apl_gemm_bf16_grouped(arr(a_ptrs), arr(b_ptrs), arr(c_ptrs), len(c_ptrs), reduce,
                                        M, N, K, lda, ldb, ldc,
                                        A.B_KN if b_layout == "kn" else A.B_NK,
                                        _DTYPE_CODE[out_dtype],
                                        A.EPI_GELU if gelu else A.EPI_NONE, None,
                                        _stream_handle(stream)))


def gelu(x: torch.Tensor, y: torch.Tensor, stream=None) -> None:
    """y = GELU(x) on the device (exact erf)."""
    check(A.lib().apl_gelu(C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), x.numel(),
                           _DTYPE_CODE[x.dtype], _stream_handle(stream)))


_gelu = gelu


def gelu_backward(dy: torch.Tensor, x: torch.Tensor, dx: torch.Tensor, stream=None) -> None:
    """dx = dy * GELU'(x) on the device."""
    check(A.lib().apl_gelu_backward(C.c_void_p(dy.data_ptr()), C.c_void_p(x.data_ptr()),
                                    C.c_void_p(dx.data_ptr()), x.numel(), _DTYPE_CODE[x.dtype],
                                    _stream_handle(stream)))


def launch_count() -> int:
    n = C.c_uint64()
    check(A.lib().apl_launch_count(C.byref(n)))
    return n.value


def gemm(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor | None = None,
         gelu: bool = False, out_dtype=torch.bfloat16, b_layout: str = "nk",
         stream=None) -> torch.Tensor:
    """out[M,N] = epi(a[M,K] . B) on the tcgen05 tensor cores (bf16 in, fp32
    accumulate). b_layout "nk": b is Bt [N,K] (nn.Linear weight); "kn": b is
    the row-major [K,N] matrix itself."""
    if a.dtype != torch.bfloat16 or b.dtype != torch.bfloat16:
        raise TypeError("gemm operands must be bf16")
    kn = b_layout == "kn"
    if a.dim() != 2 or b.dim() != 2 or a.shape[1] != (b.shape[0] if kn else b.shape[1]):
        raise ValueError("gemm wants a[M,K] and b[N,K] ('nk') or b[K,N] ('kn')")
    if a.stride(1) != 1 or b.stride(1) != 1:
        raise ValueError("operands need a unit inner stride")
    m, k = a.shape
    n = b.shape[1] if kn else b.shape[0]
    if out is None:
        out = torch.empty(m, n, dtype=out_dtype, device=a.device)
    code = _DTYPE_CODE[out.dtype]
    check(A.lib().apl_gemm_bf16(C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()),
                                C.c_void_p(out.data_ptr()), m, n, k, a.stride(0), b.stride(0),
                                out.stride(0), A.B_KN if kn else A.B_NK, code,
                                A.EPI_GELU if gelu else A.EPI_NONE, _stream_handle(stream)))
    return out


class Mesh:
    """An executing DeviceMesh.

    Mesh.local(shape)  — all mesh devices simulated as buffers on one GPU;
                         buffer lists carry num_devices tensors.
    Mesh.nccl(shape, rank, uid) — one process per GPU over NCCL; buffer
                         lists carry this rank's single shard.
    """

    def __init__(self, handle: C.c_void_p, geo: DeviceMesh, device: int):
        self._h = handle
        self.geo = geo
        self.device = device
        n, first, nl, dist = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        check(A.lib().apl_mesh_info(handle, C.byref(n), C.byref(first), C.byref(nl),
                                    C.byref(dist)))
        self.num_devices, self.first_local, self.num_local = n.value, first.value, nl.value
        self.distributed = bool(dist.value)
        self._ws = None

    @staticmethod
    def local(shape: Sequence[int], device: int = 0) -> "Mesh":
        geo = DeviceMesh.uniform(shape)
        h = C.c_void_p()
        check(A.lib().apl_mesh_create_local(C.byref(geo.c()), device, C.byref(h)))
        return Mesh(h, geo, device)

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        check(A.lib().apl_nccl_unique_id(buf))
        return bytes(buf)

    @staticmethod
    def nccl(shape: Sequence[int], rank: int, uid: bytes, device: int) -> "Mesh":
        geo = DeviceMesh.uniform(shape)
        h = C.c_void_p()
        ub = (C.c_uint8 * 128).from_buffer_copy(uid)
        check(A.lib().apl_mesh_create_nccl(C.byref(geo.c()), rank, ub, device, C.byref(h)))
        return Mesh(h, geo, device)

    @staticmethod
    def from_process_group(shape: Sequence[int]) -> "Mesh":
        """Distributed mesh over the default torch.distributed group (rank =
        mesh device index, row-major; NCCL id broadcast through the group)."""
        import torch.distributed as dist

        rank = dist.get_rank()
        obj = [Mesh.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return Mesh.nccl(shape, rank, obj[0], torch.cuda.current_device())

    def close(self) -> None:
        if self._h:
            A.lib().apl_mesh_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- failure detection (NCCL meshes) ---------------------------------------
    def health(self) -> int:
        """0 healthy, 7 (ncclInProgress) still completing, else the first
        ncclResult_t async error of any of the mesh's communicators."""
        st = C.c_int()
        check(A.lib().apl_mesh_health(self._h, C.byref(st)))
        return st.value

    def abort(self) -> None:
        """ncclCommAbort on every communicator: pending NCCL kernels return."""
        check(A.lib().apl_mesh_abort(self._h))

    def synchronize(self, stream=None, timeout_s: float = 300.0, poll_s: float = 1e-3) -> None:
        """Wait for `stream` while polling the communicators' async errors:
        raises NcclError on an async error, and on a timeout aborts the
        communicators (so the stream drains instead of hanging) and raises
        TimeoutError. Simulated meshes just synchronize."""
        import time

        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        if not self.distributed:
            s.synchronize()
            return
        from .layout import NcclError

        t0 = time.monotonic()
        while not s.query():
            st = self.health()
            if st not in (0, 7):
                self.abort()
                raise NcclError(f"NCCL async error {st} on the mesh's communicators")
            if time.monotonic() - t0 > timeout_s:
                self.abort()
                raise TimeoutError(f"mesh stream did not finish within {timeout_s} s; "
                                   "communicators aborted")
            time.sleep(poll_s)
        st = self.health()
        if st not in (0, 7):
            raise NcclError(f"NCCL async error {st} on the mesh's communicators")

    # ---- conversions ---------------------------------------------------------
    def workspace_bytes(self, path: TransformPath, meta: TensorMeta, fuse: bool = False) -> int:
        out = C.c_size_t()
        steps = path.steps_c()
        check(A.lib().apl_path_workspace_bytes(
            self._h, C.byref(path.source.c()), C.byref(path.target.c()), steps,
            len(path.steps), C.byref(meta.c()), A.FUSE_CHAIN if fuse else A.STEPWISE,
            C.byref(out)))
        return out.value

    def _workspace(self, nbytes: int) -> torch.Tensor:
        if self._ws is None or self._ws.numel() < nbytes:
            self._ws = torch.empty(max(nbytes, 256), dtype=torch.uint8,
                                   device=f"cuda:{self.device}")
        return self._ws

    def _check_bufs(self, bufs, nbytes: int, what: str) -> None:
        if len(bufs) != self.num_local:
            raise ValueError(f"{what}: expected {self.num_local} buffers, got {len(bufs)}")
        for t in bufs:
            if not t.is_cuda or not t.is_contiguous():
                raise ValueError(f"{what}: buffers must be contiguous CUDA tensors")
            if t.numel() * t.element_size() < nbytes:
                raise ValueError(f"{what}: buffer holds {t.numel() * t.element_size()} bytes, "
                                 f"needs {nbytes}")

    def run_path(self, path: TransformPath, meta: TensorMeta, inputs, outputs,
                 fuse: bool = False, stream=None) -> None:
        """Execute `path` (stepwise, or collapsed into one exchange)."""
        self._check_bufs(inputs, path.source.per_device_bytes(meta, self.geo), "inputs")
        self._check_bufs(outputs, path.target.per_device_bytes(meta, self.geo), "outputs")
        nbytes = self.workspace_bytes(path, meta, fuse)
        ws = self._workspace(nbytes)
        steps = path.steps_c()
        check(A.lib().apl_run_path(
            self._h, C.byref(path.source.c()), C.byref(path.target.c()), steps,
            len(path.steps), C.byref(meta.c()), _ptrs(inputs), _ptrs(outputs),
            C.c_void_p(ws.data_ptr()), C.c_size_t(ws.numel()),
            A.FUSE_CHAIN if fuse else A.STEPWISE, _stream_handle(stream)))

    def prepare(self, path: TransformPath, meta: TensorMeta, fuse: bool = True) -> "Conversion":
        """Validate + compile `path` once; the returned callable runs it with
        no per-call planning (and can be captured into a CUDA graph after
        its first run)."""
        return Conversion(self, path, meta, fuse)

    def run_step(self, src: ShardingSpec, step: TransformStep, meta: TensorMeta, inputs,
                 outputs, stream=None) -> None:
        path = TransformPath(src, step.result, [step])
        self.run_path(path, meta, inputs, outputs, False, stream)

    def convert(self, src: ShardingSpec, tgt: ShardingSpec, meta: TensorMeta, inputs,
                fuse: bool = True, stream=None) -> list:
        """Allocate target shards and convert `inputs` (src) into them."""
        path = find_transform_path(src, tgt, self.geo, meta)
        shape = tgt.local_shape(meta, self.geo)
        outs = [torch.empty(shape, dtype=inputs[0].dtype, device=inputs[0].device)
                for _ in range(self.num_local)]
        self.run_path(path, meta, inputs, outs, fuse, stream)
        return outs

    def exchange_traffic(self, src: ShardingSpec, tgt: ShardingSpec, meta: TensorMeta) -> dict:
        """Algorithmic bytes of the collapsed src->tgt exchange (local devices)."""
        r, w, wire = C.c_int64(), C.c_int64(), C.c_int64()
        check(A.lib().apl_exchange_traffic(self._h, C.byref(src.c()), C.byref(tgt.c()),
                                           C.byref(meta.c()), C.byref(r), C.byref(w),
                                           C.byref(wire)))
        return {"hbm_read": r.value, "hbm_write": w.value, "wire_in": wire.value}

    def exchange_engine(self, src: ShardingSpec, tgt: ShardingSpec, meta: TensorMeta) -> str:
        """'tile' (TMA tensor boxes), 'bulk' (TMA bulk ring) or 'ldg' (vectorised
        box copy) for this exchange."""
        e = C.c_int()
        check(A.lib().apl_exchange_engine(self._h, C.byref(src.c()), C.byref(tgt.c()),
                                          C.byref(meta.c()), C.byref(e)))
        return {1: "bulk", 2: "tile"}.get(e.value, "ldg")

    def sharded_matmul(self, strategy: "MatmulStrategy", a_meta: TensorMeta, b_meta: TensorMeta,
                       a_shards, b_shards, c_shards, gelu: bool = False, b_layout: str = "nk",
                       stream=None, gelu_save=None) -> None:
        """Local tcgen05 GEMM per device + partial-sum all-reduce (+ epilogue).
        b_layout "nk": each B shard stored transposed [n_local, k_local];
        "kn": the logical row-major shard [k_local, n_local]. gelu_save: one
        bf16 buffer per local device receiving the pre-activation while C
        gets GELU of it (training forward, one pass)."""
        for what, bufs in (("A", a_shards), ("B", b_shards), ("C", c_shards),
                           ("aux", gelu_save)):
            if bufs is not None and len(bufs) != self.num_local:
                raise ValueError(f"{what}: expected {self.num_local} shards")
        epi = A.EPI_GELU_SAVE if gelu_save is not None else (A.EPI_GELU if gelu else A.EPI_NONE)
        check(A.lib().apl_sharded_matmul_ex(
            self._h, C.byref(strategy.c_struct()), C.byref(a_meta.c()), C.byref(b_meta.c()),
            _ptrs(a_shards), _ptrs(b_shards), _ptrs(c_shards),
            A.B_KN if b_layout == "kn" else A.B_NK, _DTYPE_CODE[c_shards[0].dtype], epi,
            _ptrs(gelu_save) if gelu_save is not None else None, _stream_handle(stream)))

    def sharded_matmul_backward(self, strategy: "MatmulStrategy", a_meta: TensorMeta,
                                b_meta: TensorMeta, a_shards, b_shards, dc_shards,
                                da_shards=None, db_shards=None, b_layout: str = "nk",
                                gelu_aux=None, stream=None) -> None:
        """Backward of sharded_matmul: dA = dC . B^T (times GELU'(gelu_aux)
        when given) and dB = A^T . dC in B's storage layout, each summed over
        the mesh axes it is partial over (see apl_sharded_matmul_backward)."""
        n = self.num_local
        for what, bufs in (("A", a_shards), ("B", b_shards), ("dC", dc_shards),
                           ("dA", da_shards), ("dB", db_shards), ("aux", gelu_aux)):
            if bufs is not None and len(bufs) != n:
                raise ValueError(f"{what}: expected {n} shards")
        db_dtype = _DTYPE_CODE[db_shards[0].dtype] if db_shards is not None else A.F32
        check(A.lib().apl_sharded_matmul_backward(
            self._h, C.byref(strategy.c_struct()), C.byref(a_meta.c()), C.byref(b_meta.c()),
            _ptrs(a_shards) if a_shards is not None else None,
            _ptrs(b_shards) if b_shards is not None else None, _ptrs(dc_shards),
            _ptrs(da_shards) if da_shards is not None else None,
            _ptrs(db_shards) if db_shards is not None else None,
            A.B_KN if b_layout == "kn" else A.B_NK,
            A.EPI_DGELU if gelu_aux is not None else A.EPI_NONE,
            _ptrs(gelu_aux) if gelu_aux is not None else None, db_dtype, _stream_handle(stream)))

    def all_reduce(self, axes: Sequence[int], tensors, stream=None) -> None:
        if not tensors:
            return
        dt = _DTYPE_CODE[tensors[0].dtype]
        if len(tensors) != self.num_local:
            raise ValueError(f"expected {self.num_local} buffers")
        ax = (C.c_int32 * max(1, len(axes)))(*axes)
        check(A.lib().apl_all_reduce(self._h, ax, len(axes), _ptrs(tensors),
                                     tensors[0].numel(), dt, _stream_handle(stream)))


class Conversion:
    """A prepared conversion (apl_conversion_*): the path is validated and its
    exchanges compiled at construction; calling it only launches kernels /
    collectives. Keeps its Mesh alive."""

    def __init__(self, mesh: Mesh, path: TransformPath, meta: TensorMeta, fuse: bool = True):
        self.mesh, self.path, self.meta, self.fuse = mesh, path, meta, fuse
        h = C.c_void_p()
        steps = path.steps_c()
        check(A.lib().apl_conversion_create(mesh._h, C.byref(path.source.c()),
                                            C.byref(path.target.c()), steps, len(path.steps),
                                            C.byref(meta.c()),
                                            A.FUSE_CHAIN if fuse else A.STEPWISE, C.byref(h)))
        self._h = h
        n = C.c_size_t()
        check(A.lib().apl_conversion_workspace(h, C.byref(n)))
        self.workspace_bytes = n.value
        self._ws = torch.empty(max(n.value, 256), dtype=torch.uint8, device=f"cuda:{mesh.device}")
        self._in_bytes = path.source.per_device_bytes(meta, mesh.geo)
        self._out_bytes = path.target.per_device_bytes(meta, mesh.geo)
        self._ptr_cache = {}

    def _ptrs(self, ins, outs):
        key = tuple(t.data_ptr() for t in ins) + tuple(t.data_ptr() for t in outs)
        hit = self._ptr_cache.get(key)
        if hit is None:
            self.mesh._check_bufs(ins, self._in_bytes, "inputs")
            self.mesh._check_bufs(outs, self._out_bytes, "outputs")
            hit = (_ptrs(ins), _ptrs(outs))
            if len(self._ptr_cache) > 64:
                self._ptr_cache.clear()
            self._ptr_cache[key] = hit
        return hit

    def __call__(self, inputs, outputs, stream=None) -> None:
        pin, pout = self._ptrs(inputs, outputs)
        check(A.lib().apl_conversion_run(self._h, pin, pout, C.c_void_p(self._ws.data_ptr()),
                                         C.c_size_t(self._ws.numel()), _stream_handle(stream)))

    def close(self) -> None:
        if getattr(self, "_h", None):
            A.lib().apl_conversion_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---- peer memory (fused single-kernel pull exchange) ---------------------------
class _CudaArray:
    """Zero-copy view of a raw device allocation for torch.as_tensor."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (ptr, False), "version": 3, "strides": None}


class PeerMesh:
    """Distributed mesh whose transport is peer memory (CUDA IPC mapped
    pointers): every rank exports its source shard buffer, maps every other
    rank's, and a conversion is ONE kernel per rank pulling its target shard
    straight out of the peers' shards (apl_run_pull). Works between GPUs
    over NVLink/NVSwitch and between processes sharing one GPU.

    `group` is any torch.distributed process group (gloo is enough): it only
    carries the 64-byte IPC handles and the host barriers of `exchange`."""

    def __init__(self, shape: Sequence[int], rank: int, device: int, shard_bytes: int,
                 group=None):
        import torch.distributed as dist

        self.geo = DeviceMesh.uniform(shape)
        self.rank, self.device, self.group = rank, device, group
        h = C.c_void_p()
        check(A.lib().apl_mesh_create_peer(C.byref(self.geo.c()), rank, device, C.byref(h)))
        self._h = h
        ptr, handle = C.c_void_p(), (C.c_uint8 * 64)()
        check(A.lib().apl_peer_alloc(h, max(shard_bytes, 16), C.byref(ptr), handle))
        self.shard_bytes = shard_bytes
        self.local_ptr = ptr.value
        self.local = torch.as_tensor(_CudaArray(ptr.value, shard_bytes), device=f"cuda:{device}")
        # epoch flags: [ready x P][done x P] uint32, written by the peers
        P = self.geo.num_devices()
        fptr, fhandle = C.c_void_p(), (C.c_uint8 * 64)()
        check(A.lib().apl_peer_alloc(h, max(8 * P, 256), C.byref(fptr), fhandle))
        self.flags = torch.as_tensor(_CudaArray(fptr.value, 8 * P),
                                     device=f"cuda:{device}").view(torch.int32)
        self.flags.zero_()
        torch.cuda.synchronize(device)
        self.epoch = 0
        handles = [None] * P
        dist.all_gather_object(handles, (bytes(handle), bytes(fhandle)), group=group)
        self.peer_ptrs, flag_ptrs = [], []
        for r, (hb, fb) in enumerate(handles):
            if r == rank:
                self.peer_ptrs.append(ptr.value)
                flag_ptrs.append(fptr.value)
                continue
            p, q = C.c_void_p(), C.c_void_p()
            check(A.lib().apl_peer_open(h, (C.c_uint8 * 64).from_buffer_copy(hb), C.byref(p)))
            check(A.lib().apl_peer_open(h, (C.c_uint8 * 64).from_buffer_copy(fb), C.byref(q)))
            self.peer_ptrs.append(p.value)
            flag_ptrs.append(q.value)
        self._table = (C.c_void_p * len(self.peer_ptrs))(*self.peer_ptrs)
        self._flag_ptrs = flag_ptrs
        self._all_flags = (C.c_void_p * P)(*flag_ptrs)
        self._counter = torch.zeros(4, dtype=torch.int32, device=f"cuda:{device}")
        self._peers = {}           # (src, tgt, shape, eb) -> (senders, readers)
        self._last_readers = None  # done slots wait_readers() waits on
        others = [q for q in range(P) if q != rank]
        self._peer_flags = (C.c_void_p * len(others))(*[flag_ptrs[q] for q in others])
        self._n_others = len(others)
        self._ready_slots = (C.c_int32 * max(1, len(others)))(*others)
        self._done_slots = (C.c_int32 * max(1, len(others)))(*[P + q for q in others])
        self.timeout_ms = 60000

    def shard(self, shape, dtype) -> torch.Tensor:
        """This rank's exported source shard as a typed tensor view."""
        n = 1
        for e in shape:
            n *= e
        nbytes = n * torch.empty((), dtype=dtype).element_size()
        if nbytes > self.shard_bytes:
            raise ValueError("shard larger than the exported buffer")
        return self.local[:nbytes].view(dtype).view(*shape)

    def pull(self, src: ShardingSpec, tgt: ShardingSpec, meta: TensorMeta, out: torch.Tensor,
             stream=None) -> None:
        """Stream-ordered fused exchange into `out` (no host synchronisation)."""
        if src.per_device_bytes(meta, self.geo) > self.shard_bytes:
            raise ValueError("source shard larger than the exported buffer")
        if out.numel() * out.element_size() < tgt.per_device_bytes(meta, self.geo):
            raise ValueError("output too small")
        check(A.lib().apl_run_pull(self._h, C.byref(src.c()), C.byref(tgt.c()), C.byref(meta.c()),
                                   self._table, C.c_void_p(out.data_ptr()), _stream_handle(stream)))

    def exchange(self, src: ShardingSpec, tgt: ShardingSpec, meta: TensorMeta,
                 out: torch.Tensor) -> None:
        """pull() bracketed by host barriers: every rank's source is complete
        before anyone reads it and stays untouched until everyone has read."""
        import torch.distributed as dist

        torch.cuda.synchronize(self.device)
        dist.barrier(group=self.group)
        self.pull(src, tgt, meta, out)
        torch.cuda.synchronize(self.device)
        dist.barrier(group=self.group)

    def exchange_peers(self, src: ShardingSpec, tgt: ShardingSpec, meta: TensorMeta):
        """(ranks this rank reads from, ranks that read this rank's source)."""
        key = (src.to_string(), tgt.to_string(), tuple(meta.shape), meta.dtype_bytes)
        hit = self._peers.get(key)
        if hit is None:
            P = self.geo.num_devices()
            sa, ra = (C.c_int32 * P)(), (C.c_int32 * P)()
            ns, nr = C.c_int(), C.c_int()
            check(A.lib().apl_exchange_peers(self._h, C.byref(src.c()), C.byref(tgt.c()),
                                             C.byref(meta.c()), sa, C.byref(ns), ra,
                                             C.byref(nr)))
            hit = self._peers[key] = (list(sa[:ns.value]), list(ra[:nr.value]))
        return hit

    def exchange_async(self, src: ShardingSpec, tgt: ShardingSpec, meta: TensorMeta,
                       out: torch.Tensor, stream=None, fused: bool | None = None) -> int:
        """Stream-ordered exchange synchronised on the device, no host
        barrier. fused (default; APL_PEER_FUSED=0 selects the 4-launch form):
        ONE kernel announces this rank's source (ready flag at every peer),
        acquires the ready flags of the ranks it actually reads from, pulls,
        and its last CTA announces that this rank finished reading
        (apl_run_pull_sync). Unfused: flag-store kernel, flag-wait kernel on
        every peer, pull kernel, flag-store kernel. Returns the epoch. Call
        wait_readers() before overwriting the exported source."""
        if fused is None:
            import os

            fused = os.environ.get("APL_PEER_FUSED", "1") != "0"
        self.epoch += 1
        e, r, P = self.epoch, self.rank, self.geo.num_devices()
        sh = _stream_handle(stream)
        lib = A.lib()
        if fused:
            if src.per_device_bytes(meta, self.geo) > self.shard_bytes:
                raise ValueError("source shard larger than the exported buffer")
            if out.numel() * out.element_size() < tgt.per_device_bytes(meta, self.geo):
                raise ValueError("output too small")
            _, readers = self.exchange_peers(src, tgt, meta)
            sync = A.PeerSyncC(self._all_flags, self.flags.data_ptr(), self._counter.data_ptr(),
                               e, self.timeout_ms)
            check(lib.apl_run_pull_sync(self._h, C.byref(src.c()), C.byref(tgt.c()),
                                        C.byref(meta.c()), self._table,
                                        C.c_void_p(out.data_ptr()), C.byref(sync), sh))
            self._last_readers = readers
            return e
        check(lib.apl_peer_flags_store(self._peer_flags, self._n_others, r, e, sh))
        check(lib.apl_peer_flags_wait(C.c_void_p(self.flags.data_ptr()), self._ready_slots,
                                      self._n_others, e, self.timeout_ms, sh))
        self.pull(src, tgt, meta, out, stream=stream)
        check(lib.apl_peer_flags_store(self._peer_flags, self._n_others, P + r, e, sh))
        self._last_readers = None
        return e

    def push_output(self, nbytes: int):
        """The exported output buffer push exchanges of this size write into:
        (this rank's uint8 tensor, [rank q's buffer mapped here for every q]).
        Collective on the first use of a size (shared_buffer)."""
        key = -(-max(nbytes, 16) // 256) * 256
        bufs = self.__dict__.setdefault("_push_bufs", {})
        if key not in bufs:
            local, ptrs = self.shared_buffer(key)
            bufs[key] = (local, ptrs, (C.c_void_p * len(ptrs))(*ptrs))
        return bufs[key]

    def push_async(self, src: ShardingSpec, tgt: ShardingSpec, meta: TensorMeta,
                   x: torch.Tensor, stream=None) -> torch.Tensor:
        """The exchange as a PUSH (apl_run_push_sync): ONE kernel stores every
        piece of this rank's source `x` (any local tensor) straight into the
        receivers' exported outputs, after they announced this epoch, and
        marks done at every peer after a system-scope fence; then this rank
        waits (stream-ordered) for done of the ranks that write to it.
        Returns this rank's output: a view of the push buffer, valid in
        stream order until the next push of the same size. The source is
        never read remotely, so it may be overwritten right after."""
        if x.numel() * x.element_size() < src.per_device_bytes(meta, self.geo):
            raise ValueError("source smaller than the shard")
        nbytes = tgt.per_device_bytes(meta, self.geo)
        local, _, table = self.push_output(nbytes)
        self.epoch += 1
        e, P = self.epoch, self.geo.num_devices()
        sh = _stream_handle(stream)
        senders, _ = self.exchange_peers(src, tgt, meta)
        sync = A.PeerSyncC(self._all_flags, self.flags.data_ptr(), self._counter.data_ptr(), e,
                           self.timeout_ms)
        check(A.lib().apl_run_push_sync(self._h, C.byref(src.c()), C.byref(tgt.c()),
                                        C.byref(meta.c()), C.c_void_p(x.data_ptr()), table,
                                        C.byref(sync), sh))
        if senders:
            slots = (C.c_int32 * len(senders))(*[P + q for q in senders])
            check(A.lib().apl_peer_flags_wait(C.c_void_p(self.flags.data_ptr()), slots,
                                              len(senders), e, self.timeout_ms, sh))
        self._last_readers = []  # nobody reads this rank's source remotely
        return local[:nbytes]

    def shared_buffer(self, nbytes: int):
        """Collective: allocate and export a device buffer on every rank and
        map every peer's. Returns (this rank's buffer as a uint8 tensor,
        [device pointer of rank q's buffer, mapped here, for every q])."""
        import torch.distributed as dist

        ptr, handle = C.c_void_p(), (C.c_uint8 * 64)()
        check(A.lib().apl_peer_alloc(self._h, max(nbytes, 16), C.byref(ptr), handle))
        local = torch.as_tensor(_CudaArray(ptr.value, nbytes), device=f"cuda:{self.device}")
        handles = [None] * self.geo.num_devices()
        dist.all_gather_object(handles, bytes(handle), group=self.group)
        ptrs = []
        for q, hb in enumerate(handles):
            if q == self.rank:
                ptrs.append(ptr.value)
                continue
            p = C.c_void_p()
            check(A.lib().apl_peer_open(self._h, (C.c_uint8 * 64).from_buffer_copy(hb), C.byref(p)))
            ptrs.append(p.value)
        return local, ptrs

    def axis_group(self, axes) -> list:
        """Ranks sharing this rank's coordinates off `axes`, in the order of
        their mixed-radix coordinate on `axes` (the reference's replica-group
        order, cluster.hpp:56; row-major rank <-> coordinate)."""
        shape = list(self.geo.shape)
        coord, r = [], self.rank
        for n in reversed(shape):
            coord.append(r % n)
            r //= n
        coord.reverse()
        axes = sorted(axes)
        members = []
        for idx in itertools.product(*[range(shape[a]) for a in axes]):
            c = list(coord)
            for a, v in zip(axes, idx):
                c[a] = v
            rank = 0
            for e, n in zip(c, shape):
                rank = rank * n + e
            members.append(rank)
        return members

    def matmul_allreduce(self, a: torch.Tensor, b: torch.Tensor, out_dtype=torch.bfloat16,
                         b_layout: str = "kn", stream=None, axes=None) -> torch.Tensor:
        """Split-k matmul over the ranks of this rank's `axes` group (None:
        every mesh axis) with its all-reduce fused in (Megatron fc2, reference
        split-k strategies, intraop.cpp:141-234 with the partial-sum
        all-reduce over reduce_axes of planner.cpp:263-282):
        C = sum_{r in group} A_r . B_r on every group member, bit-identical
        replicas; groups that differ off `axes` run independently.

        Two kernels instead of GEMM + a collective: the GEMM's epilogue stores
        each row block of its fp32 partial straight into the owning member's
        staging slab (reduce-scatter traffic overlapping the MMAs), then each
        owner sums its slabs and stores its rows into every member's output
        (the all-gather as peer stores); device-side epoch flags, exchanged
        only within the group, order them. Returns this rank's exported
        output (valid until the next call with the same shape and axes)."""
        axes = tuple(range(self.geo.rank())) if axes is None else tuple(sorted(axes))
        members = self.axis_group(axes)
        P, r, me = len(members), self.rank, members.index(self.rank)
        if P > 8:
            raise ValueError("fused peer all-reduce groups hold at most 8 ranks")
        M, K = a.shape
        N = b.shape[1] if b_layout == "kn" else b.shape[0]
        eb = torch.empty((), dtype=out_dtype).element_size()
        if M % P or (M // P) % 128:
            raise ValueError("M / group size must be a multiple of 128")
        rpo = M // P
        key = (M, N, out_dtype, axes)
        bufs = getattr(self, "_ar_bufs", None)
        if bufs is None:
            bufs = self._ar_bufs = {}
        if key not in bufs:
            staging, staging_peers = self.shared_buffer(P * rpo * N * 4)
            c_local, c_peers = self.shared_buffer(M * N * eb)
            slabs = (C.c_void_p * P)(*[staging_peers[q] + me * rpo * N * 4 for q in members])
            outs = (C.c_void_p * P)(*[c_peers[q] + me * rpo * N * eb for q in members])
            others = [q for q in members if q != r]
            flags = (C.c_void_p * max(1, len(others)))(*[self._flag_ptrs[q] for q in others])
            Pm = self.geo.num_devices()
            ready = (C.c_int32 * max(1, len(others)))(*others)
            done = (C.c_int32 * max(1, len(others)))(*[Pm + q for q in others])
            bufs[key] = (staging, c_local.view(out_dtype).view(M, N), slabs, outs, flags,
                         len(others), ready, done)
        staging, c_out, slabs, outs, flags, n_others, ready, done = bufs[key]
        self.epoch += 1
        e = self.epoch
        self._last_readers = None  # conservative: wait_readers waits on every rank
        sh = _stream_handle(stream)
        lib = A.lib()
        Pm = self.geo.num_devices()
        check(lib.apl_peer_gemm_scatter(C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()), slabs, P,
                                        M, N, K, a.stride(0), b.stride(0),
                                        A.B_KN if b_layout == "kn" else A.B_NK, sh))
        if n_others:
            check(lib.apl_peer_flags_store(flags, n_others, r, e, sh))
            check(lib.apl_peer_flags_wait(C.c_void_p(self.flags.data_ptr()), ready, n_others, e,
                                          self.timeout_ms, sh))
        check(lib.apl_peer_reduce_gather(C.c_void_p(staging.data_ptr()), P, rpo * N, outs, P,
                                         _DTYPE_CODE[out_dtype], sh))
        if n_others:
            check(lib.apl_peer_flags_store(flags, n_others, Pm + r, e, sh))
            check(lib.apl_peer_flags_wait(C.c_void_p(self.flags.data_ptr()), done, n_others, e,
                                          self.timeout_ms, sh))
        # ranks outside the group did not touch this rank's flags this epoch:
        # raise their slots too so wait_readers / later epochs see a uniform epoch
        outside = [q for q in range(Pm) if q not in members]
        if outside:
            check(lib.apl_peer_flags_store(
                (C.c_void_p * len(outside))(*[self._flag_ptrs[q] for q in outside]), len(outside),
                r, e, sh))
            check(lib.apl_peer_flags_store(
                (C.c_void_p * len(outside))(*[self._flag_ptrs[q] for q in outside]), len(outside),
                Pm + r, e, sh))
        return c_out

    def sharded_matmul(self, strategy: "MatmulStrategy", a: torch.Tensor, b: torch.Tensor,
                       gelu: bool = False, b_layout: str = "kn", stream=None) -> torch.Tensor:
        """This rank's part of a sharded-matmul strategy on the peer mesh:
        strategies without a partial sum are one local tcgen05 GEMM on the
        shards (GELU fused); partial-sum strategies run as the fused GEMM +
        all-reduce over peer memory within each reduce_axes group
        (matmul_allreduce), GELU (if any) applied after the sum."""
        if not strategy.partial_sum:
            return gemm(a, b, gelu=gelu, b_layout=b_layout, stream=stream)
        c = self.matmul_allreduce(a, b, b_layout=b_layout, stream=stream,
                                  axes=tuple(strategy.reduce_axes))
        if gelu:
            _gelu(c, c, stream=stream)  # (the `gelu` argument shadows the module function)
        return c

    def exchange_traffic(self, src: ShardingSpec, tgt: ShardingSpec, meta: TensorMeta) -> dict:
        """This rank's bytes of the src->tgt exchange (wire_in = bytes pulled
        from peers)."""
        return Mesh.exchange_traffic(self, src, tgt, meta)

    def wait_readers(self, stream=None) -> None:
        """Stream-ordered: block until every peer finished reading this
        rank's source of the last epoch (then it may be overwritten)."""
        if self.epoch == 0:
            return
        if self._last_readers is not None:  # only the ranks that read it
            if not self._last_readers:
                return
            P = self.geo.num_devices()
            slots = (C.c_int32 * len(self._last_readers))(*[P + q for q in self._last_readers])
            check(A.lib().apl_peer_flags_wait(C.c_void_p(self.flags.data_ptr()), slots,
                                              len(self._last_readers), self.epoch,
                                              self.timeout_ms, _stream_handle(stream)))
            return
        check(A.lib().apl_peer_flags_wait(C.c_void_p(self.flags.data_ptr()), self._done_slots,
                                          self._n_others, self.epoch, self.timeout_ms,
                                          _stream_handle(stream)))

    def close(self) -> None:
        if getattr(self, "_h", None):
            A.lib().apl_mesh_destroy(self._h)
            self._h = None
