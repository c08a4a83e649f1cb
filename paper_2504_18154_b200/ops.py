"""Op-level wrappers (include/ecoserve_ops.h) over torch CUDA tensors."""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib as L


def _s(stream=None):
    return C.c_void_p(torch.cuda.current_stream().cuda_stream if stream is None else stream)


def gemm(A: torch.Tensor, B: torch.Tensor, out_dtype=torch.float32, bn: int = 256) -> torch.Tensor:
    m, k = A.shape
    n = B.shape[0]
    out = torch.empty(m, n, dtype=out_dtype, device=A.device)
    L.check(L.load().ecoserve_op_gemm(A.data_ptr(), B.data_ptr(), m, n, k, 0 if out_dtype == torch.float32 else 1,
                                      out.data_ptr(), bn, _s()))
    return out


def gemm_swap(W: torch.Tensor, X: torch.Tensor, splits: int = 1, bn: int = 64) -> torch.Tensor:
    m, k = W.shape
    n = X.shape[0]
    ws = torch.empty(splits, n, m, dtype=torch.float32, device=W.device)
    out = torch.empty(n, m, dtype=torch.float32, device=W.device)
    L.check(L.load().ecoserve_op_gemm_swap(W.data_ptr(), X.data_ptr(), m, n, k, splits, ws.data_ptr(), out.data_ptr(),
                                           bn, _s()))
    return out


def gemm_swap_bf16(W: torch.Tensor, X: torch.Tensor, splits: int = 1, bn: int = 64,
                   check_counters: bool = False) -> torch.Tensor:
    """out bf16 [n][m] = X W^T through the in-kernel split-K reduction path."""
    m, k = W.shape
    n = X.shape[0]
    part = torch.empty(splits, n, m, dtype=torch.float32, device=W.device)
    cnt = torch.zeros(((m + 127) // 128) * ((n + bn - 1) // bn), dtype=torch.int32, device=W.device)
    out = torch.empty(n, m, dtype=torch.bfloat16, device=W.device)
    L.check(L.load().ecoserve_op_gemm_swap_bf16(W.data_ptr(), X.data_ptr(), m, n, k, splits, part.data_ptr(),
                                                cnt.data_ptr(), out.data_ptr(), bn, _s()))
    if check_counters:
        assert int(cnt.abs().sum()) == 0, "split-K counters must be left at zero"
    return out


def gemm_decode(W: torch.Tensor, X: torch.Tensor, r: int = 2, splits: int = 1, bn: int = 128) -> torch.Tensor:
    """out f32 [n][m] = X W^T through the engine's decode-GEMM configuration."""
    m, k = W.shape
    n = X.shape[0]
    ws = torch.empty(max(splits, 1), n, m, dtype=torch.float32, device=W.device) if splits > 1 else None
    out = torch.empty(n, m, dtype=torch.float32, device=W.device)
    L.check(L.load().ecoserve_op_gemm_decode(W.data_ptr(), X.data_ptr(), m, n, k, r, splits,
                                             ws.data_ptr() if ws is not None else None, out.data_ptr(), bn, _s()))
    return out


def gemm_decode_balanced(W: torch.Tensor, X: torch.Tensor, max_slots: int = 8, bn: int = 128):
    """out f32 [n][m] = X W^T with the balanced split-K (equal K-block chunks per CTA);
    returns (out, chunk length)."""
    import ctypes
    m, k = W.shape
    n = X.shape[0]
    ws = torch.empty(max_slots, n, m, dtype=torch.float32, device=W.device)
    out = torch.empty(n, m, dtype=torch.float32, device=W.device)
    chunk = ctypes.c_int32(0)
    L.check(L.load().ecoserve_op_gemm_decode_balanced(W.data_ptr(), X.data_ptr(), m, n, k, max_slots, ws.data_ptr(),
                                                      out.data_ptr(), bn, ctypes.byref(chunk), _s()))
    return out, chunk.value


def gemm_cluster(W: torch.Tensor, X: torch.Tensor, splits: int, bn: int = 128) -> torch.Tensor:
    """out f32 [n][m] = X W^T, K split over a thread-block cluster, reduced in DSMEM."""
    m, k = W.shape
    n = X.shape[0]
    out = torch.empty(n, m, dtype=torch.float32, device=W.device)
    L.check(L.load().ecoserve_op_gemm_cluster(W.data_ptr(), X.data_ptr(), m, n, k, splits, out.data_ptr(), bn, _s()))
    return out


def lm_argmax(W: torch.Tensor, X: torch.Tensor) -> torch.Tensor:
    V, k = W.shape
    n = X.shape[0]
    parts = (V + 127) // 128
    wv = torch.empty(n, parts, dtype=torch.float32, device=W.device)
    wi = torch.empty(n, parts, dtype=torch.int32, device=W.device)
    tok = torch.empty(n, dtype=torch.int32, device=W.device)
    L.check(L.load().ecoserve_op_lm_argmax(W.data_ptr(), X.data_ptr(), V, n, k, wv.data_ptr(), wi.data_ptr(),
                                           tok.data_ptr(), _s()))
    return tok


def rmsnorm(x: torch.Tensor, gamma: torch.Tensor, eps: float, rows=None) -> torch.Tensor:
    n = x.shape[0] if rows is None else rows.shape[0]
    H = x.shape[1]
    out = torch.empty(n, H, dtype=torch.bfloat16, device=x.device)
    L.check(L.load().ecoserve_op_rmsnorm(x.data_ptr(), None if rows is None else rows.data_ptr(), gamma.data_ptr(),
                                         out.data_ptr(), n, H, eps, _s()))
    return out


def _offsets(ctx_off):
    if ctx_off is None:
        return None, None
    off = np.ascontiguousarray(ctx_off, dtype=np.int32)
    return off, off.ctypes.data_as(L.PI32)


def attention_prefill(q, pool, num_blocks, n_heads, n_kv, head_dim, cu_seqlens, block_tables, ctx_off=None):
    """ctx_off: per-sequence cached tokens before the chunk (chunked prefill), or None."""
    T = q.shape[0]
    out = torch.empty(T, n_heads * head_dim, dtype=torch.bfloat16, device=q.device)
    cu = np.ascontiguousarray(cu_seqlens, dtype=np.int32)
    n_seq = len(cu) - 1
    off, poff = _offsets(ctx_off)
    L.check(L.load().ecoserve_op_attention_prefill(q.data_ptr(), pool.data_ptr(), num_blocks, n_heads, n_kv, head_dim,
                                                   cu.ctypes.data_as(L.PI32), n_seq, block_tables.data_ptr(),
                                                   block_tables.shape[1], out.data_ptr(), _s(), poff))
    return out


def attention_prefill_tc(q, pool, num_blocks, n_heads, n_kv, cu_seqlens, block_tables, ctx_off=None):
    T = q.shape[0]
    out = torch.empty(T, n_heads * 128, dtype=torch.bfloat16, device=q.device)
    cu = np.ascontiguousarray(cu_seqlens, dtype=np.int32)
    off, poff = _offsets(ctx_off)
    L.check(L.load().ecoserve_op_attention_prefill_tc(q.data_ptr(), pool.data_ptr(), num_blocks, n_heads, n_kv,
                                                      cu.ctypes.data_as(L.PI32), len(cu) - 1, block_tables.data_ptr(),
                                                      block_tables.shape[1], out.data_ptr(), _s(), poff))
    return out


def attention_decode(q, pool, n_heads, n_kv, head_dim, ctx_lens, block_tables, n_splits, blocks_per_split,
                     use_tma=False):
    """use_tma (head_dim 128): K / V staged by TMA, the engine's path."""
    B = q.shape[0]
    out = torch.empty(B, n_heads * head_dim, dtype=torch.bfloat16, device=q.device)
    ws = torch.empty(B * n_heads * n_splits * (head_dim + 2), dtype=torch.float32, device=q.device)
    L.check(L.load().ecoserve_op_attention_decode(q.data_ptr(), pool.data_ptr(), n_heads, n_kv, head_dim,
                                                  ctx_lens.data_ptr(), B, block_tables.data_ptr(),
                                                  block_tables.shape[1], n_splits, blocks_per_split, ws.data_ptr(),
                                                  out.data_ptr(), _s(), 1 if use_tma else 0))
    return out


def attention_decode_sk(q, pool, n_heads, n_kv, head_dim, ctx_lens, block_tables):
    """Persistent stream-K decode attention (head_dim 128); ctx_lens: host int sequence."""
    import numpy as np
    B = q.shape[0]
    out = torch.empty(B, n_heads * head_dim, dtype=torch.bfloat16, device=q.device)
    ws = torch.empty(B * n_heads * 64 * (head_dim + 2), dtype=torch.float32, device=q.device)
    cnt = torch.zeros(B * n_kv, dtype=torch.int32, device=q.device)
    meta = torch.empty(2 * B + 1, dtype=torch.int32, device=q.device)
    ctx = np.ascontiguousarray(ctx_lens, dtype=np.int32)
    L.check(L.load().ecoserve_op_attention_decode_sk(q.data_ptr(), pool.data_ptr(), n_heads, n_kv, head_dim,
                                                     ctx.ctypes.data_as(L.PI32), B, block_tables.data_ptr(),
                                                     block_tables.shape[1], ws.data_ptr(), cnt.data_ptr(),
                                                     meta.data_ptr(), out.data_ptr(), _s()))
    assert int(cnt.abs().sum()) == 0, "item counters must be left at zero"
    return out
