"""Transformer-block node kinds on one shard (apl_embedding_lookup, apl_layernorm,
apl_softmax, apl_transpose, apl_scale, apl_add, apl_mask_not; block_ops.cu).

The non-GEMM kinds of the reference's gpt_block graph (graph_ir.cpp:40-46,
shape rules graph_ir.cpp:240-345). The reference's strategies keep all of
them local (intraop.cpp:280-450), so each call works on one device's shard
and never communicates. Tensors in, tensors out; no torch compute, no fallback.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _capi as A
from .layout import check
from .runtime import _DTYPE_CODE, _stream_handle


def _p(t: torch.Tensor | None) -> C.c_void_p:
    return C.c_void_p(t.data_ptr() if t is not None else None)


def embedding(ids: torch.Tensor, table: torch.Tensor, out: torch.Tensor, stream=None) -> None:
    """out[..., :] = table[ids[...], :]; ids int64, table [vocab, width]."""
    if ids.dtype != torch.int64:
        raise TypeError("ids must be int64")
    check(A.lib().apl_embedding_lookup(_p(ids), ids.numel(), _p(table), table.shape[0],
                                       table.shape[1], table.element_size(), _p(out),
                                       _stream_handle(stream)))


def embedding_blocks(ids: torch.Tensor, block_ptrs, vocab_blocks: int, hidden_blocks: int,
                     vocab: int, width: int, col_begin: int, out: torch.Tensor,
                     stream=None) -> None:
    """out = table[ids, col_begin : col_begin + out.shape[-1]] with the table
    given as its owners' blocks (row-major [vocab_blocks x hidden_blocks]
    device addresses): the table's all-gather fused into the lookup."""
    if ids.dtype != torch.int64:
        raise TypeError("ids must be int64")
    arr = (C.c_void_p * len(block_ptrs))(*block_ptrs)
    check(A.lib().apl_embedding_lookup_blocks(_p(ids), ids.numel(), arr, vocab_blocks,
                                              hidden_blocks, vocab, width, col_begin,
                                              out.shape[-1], out.element_size(), _p(out),
                                              _stream_handle(stream)))


def layernorm(x: torch.Tensor, gamma: torch.Tensor | None, beta: torch.Tensor | None,
              y: torch.Tensor, eps: float = 1e-5, stream=None) -> None:
    w = x.shape[-1]
    check(A.lib().apl_layernorm(_p(x), _p(gamma), _p(beta), _p(y), x.numel() // w, w, eps,
                                _DTYPE_CODE[x.dtype], _stream_handle(stream)))


def softmax(x: torch.Tensor, y: torch.Tensor, stream=None) -> None:
    """Softmax over the last dim."""
    w = x.shape[-1]
    check(A.lib().apl_softmax(_p(x), _p(y), x.numel() // w, w, _DTYPE_CODE[x.dtype],
                              _stream_handle(stream)))


def masked_softmax(x: torch.Tensor, y: torch.Tensor, alpha: float = 1.0,
                   mask: torch.Tensor | None = None, fill: float = 0.0, stream=None) -> None:
    """y = softmax(alpha * x + fill * mask) over the last dim, one pass."""
    if mask is not None and (mask.dtype != torch.uint8 or mask.numel() != x.numel()):
        raise TypeError("mask must be uint8 of x's size")
    w = x.shape[-1]
    check(A.lib().apl_softmax_ex(_p(x), _p(y), x.numel() // w, w, alpha, _p(mask), fill,
                                 _DTYPE_CODE[x.dtype], _stream_handle(stream)))


def transpose_last2(x: torch.Tensor, y: torch.Tensor, stream=None) -> None:
    """y = x with its last two dims swapped (perm [..., -1, -2])."""
    r, c = x.shape[-2], x.shape[-1]
    check(A.lib().apl_transpose(_p(x), _p(y), x.numel() // max(1, r * c), r, c,
                                x.element_size(), _stream_handle(stream)))


def permute(x: torch.Tensor, y: torch.Tensor, perm, stream=None) -> None:
    """y = x.permute(perm) materialised (row-major), any permutation of rank
    <= 8: the graph's general transpose (apl_permute)."""
    perm = [int(p) for p in perm]
    if sorted(perm) != list(range(x.dim())) or list(y.shape) != [x.shape[p] for p in perm]:
        raise ValueError(f"bad permutation {perm} for {tuple(x.shape)} -> {tuple(y.shape)}")
    I64 = C.c_int64 * max(1, x.dim())
    check(A.lib().apl_permute(_p(x), _p(y), x.dim(), I64(*x.shape), I64(*perm),
                              x.element_size(), _stream_handle(stream)))


def _axis_split(shape, axis):
    axis = axis % len(shape)
    outer = 1
    for e in shape[:axis]:
        outer *= e
    inner = 1
    for e in shape[axis + 1:]:
        inner *= e
    return outer, shape[axis], inner


def softmax_axis(x: torch.Tensor, y: torch.Tensor, axis: int, stream=None) -> None:
    """Softmax over any axis (the last one takes the row kernels)."""
    o, n, i = _axis_split(tuple(x.shape), axis)
    check(A.lib().apl_softmax_axis(_p(x), _p(y), o, n, i, _DTYPE_CODE[x.dtype],
                                   _stream_handle(stream)))


def softmax_axis_backward(y: torch.Tensor, dy: torch.Tensor, dx: torch.Tensor, axis: int,
                          alpha: float = 1.0, stream=None) -> None:
    o, n, i = _axis_split(tuple(y.shape), axis)
    check(A.lib().apl_softmax_axis_backward(_p(y), _p(dy), _p(dx), o, n, i, alpha,
                                            _DTYPE_CODE[y.dtype], _stream_handle(stream)))


def scale(x: torch.Tensor, y: torch.Tensor, alpha: float, stream=None) -> None:
    check(A.lib().apl_scale(_p(x), _p(y), x.numel(), alpha, _DTYPE_CODE[x.dtype],
                            _stream_handle(stream)))


def add(a: torch.Tensor, b: torch.Tensor, y: torch.Tensor, alpha: float = 1.0,
        stream=None) -> None:
    """y = a + alpha * b; b of a's dtype, or a uint8 0/1 mask."""
    mask = b.dtype == torch.uint8
    if not mask and b.dtype != a.dtype:
        raise TypeError("b must have a's dtype or be a uint8 mask")
    check(A.lib().apl_add(_p(a), _p(b), 1 if mask else 0, _p(y), a.numel(), alpha,
                          _DTYPE_CODE[a.dtype], _stream_handle(stream)))


def mask_not(x: torch.Tensor, y: torch.Tensor, stream=None) -> None:
    """y = !x on a uint8 mask."""
    check(A.lib().apl_mask_not(_p(x), _p(y), x.numel(), _stream_handle(stream)))


# ---- backward -----------------------------------------------------------------
def layernorm_backward(x: torch.Tensor, gamma: torch.Tensor | None, dy: torch.Tensor,
                       dx: torch.Tensor, dgamma: torch.Tensor | None = None,
                       dbeta: torch.Tensor | None = None, eps: float = 1e-5,
                       stream=None) -> None:
    """dx of a layernorm; dgamma / dbeta (fp32) are ACCUMULATED into."""
    w = x.shape[-1]
    rows = x.numel() // w
    stats, nbytes = None, 0
    if dgamma is not None or dbeta is not None:
        n = C.c_size_t()
        check(A.lib().apl_layernorm_backward_scratch(rows, w, C.byref(n)))
        stats = torch.empty((n.value + 15) // 16 * 4, dtype=torch.float32, device=x.device)
        nbytes = stats.numel() * 4
    check(A.lib().apl_layernorm_backward_ex(_p(x), _p(gamma), _p(dy), _p(dx), _p(dgamma),
                                            _p(dbeta), _p(stats), nbytes, rows, w, eps,
                                            _DTYPE_CODE[x.dtype], _stream_handle(stream)))


def softmax_backward(y: torch.Tensor, dy: torch.Tensor, dx: torch.Tensor, alpha: float = 1.0,
                     stream=None) -> None:
    w = y.shape[-1]
    check(A.lib().apl_softmax_backward(_p(y), _p(dy), _p(dx), y.numel() // w, w, alpha,
                                       _DTYPE_CODE[y.dtype], _stream_handle(stream)))


def embedding_backward(ids: torch.Tensor, dy: torch.Tensor, dtable: torch.Tensor,
                       stream=None) -> None:
    """dtable[ids] += dy (dtable fp32 [vocab, width], accumulated)."""
    if dtable.dtype != torch.float32:
        raise TypeError("dtable must be fp32")
    check(A.lib().apl_embedding_backward(_p(ids), ids.numel(), _p(dy), _p(dtable),
                                         dtable.shape[0], dtable.shape[1],
                                         _DTYPE_CODE[dy.dtype], _stream_handle(stream)))


def embedding_backward_block(ids: list, dys: list, dblock: torch.Tensor, v0: int, c0: int,
                             stream=None) -> None:
    """dblock += the rows of every (ids[s], dys[s]) source whose id lies in
    [v0, v0 + dblock.shape[0]), columns [c0, c0 + dblock.shape[1]) of dy:
    one owner block of a table gradient, reduce-scatter fused."""
    P = C.c_void_p
    n = ids[0].numel()
    if any(i.numel() != n for i in ids):
        raise ValueError("every source holds the same number of ids")
    check(A.lib().apl_embedding_backward_block(
        (P * len(ids))(*[i.data_ptr() for i in ids]), (P * len(dys))(*[d.data_ptr() for d in dys]),
        len(ids), n, dys[0].shape[-1], _p(dblock), v0, dblock.shape[0], c0, dblock.shape[1],
        _DTYPE_CODE[dys[0].dtype], _stream_handle(stream)))


def bmm(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor, a_t: bool = False,
        b_t: bool = False, stream=None) -> None:
    """out[i] = op(a[i]) . op(b[i]) for every batch i on the tcgen05 tensor
    cores (one grouped launch); op = transpose when a_t / b_t. bf16 in, fp32
    accumulate, out bf16 or fp32."""
    nb = a.shape[0]
    M = a.shape[2] if a_t else a.shape[1]
    K = a.shape[1] if a_t else a.shape[2]
    N = b.shape[1] if b_t else b.shape[2]
    ea, eb, eo = a.element_size(), b.element_size(), out.element_size()
    P = C.c_void_p
    arr = lambda xs: (P * len(xs))(*xs)  # noqa: E731
    check(A.lib().apl_gemm_bf16_grouped_ex(
        arr([a.data_ptr() + i * a[0].numel() * ea for i in range(nb)]),
        arr([b.data_ptr() + i * b[0].numel() * eb for i in range(nb)]),
        arr([out.data_ptr() + i * M * N * eo for i in range(nb)]), nb, M, N, K,
        a.shape[2], b.shape[2], N, 1 if a_t else 0, 0 if b_t else 1, _DTYPE_CODE[out.dtype],
        _stream_handle(stream)))
