"""ORACLE (test infrastructure only) -- fp64 Llama-family decoder, SURVEY 8(c) C1-C4.

What the PaDG instance computes: PaDG changes *when* prefill and decode run
(Sec. 3.2.1), never *what* they compute, so the oracle is
the plain definition of the transformer the paper evaluates:

* Eq. 1: Q = X Wq^T, K = X Wk^T, V = X Wv^T (GQA, reading A5).
* Eq. 2: softmax(Q K^T / sqrt(d_k)) V, causal per sequence (A2).
* Eq. 3: FFN, read as Llama SwiGLU W_down(silu(x W_g^T) * x W_u^T)
  without biases (reading A1), after RMSNorm ("layer normalization",
  reading A4), with RoPE rotate-half (reading A3).
* Fig. 2: prefill emits token 0 and initializes the KV cache; each
  decode step feeds back one token (greedy argmax, lowest index on ties, A6).

Everything is float64; weights are the bf16 values from ``synthetic.weights``.
No blocking, fusion or reordering beyond the definitions.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

BLOCK_TOKENS = 64  # KV block size (SURVEY 8 notation; PagedAttention P:824)


# ---------------------------------------------------------------- primitives
def rmsnorm(x: np.ndarray, gamma: np.ndarray, eps: float) -> np.ndarray:
    """x / sqrt(mean(x^2) + eps) * gamma, row-wise (readings A1, A4)."""
    return x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps) * gamma


def rope_cos_sin(positions: np.ndarray, head_dim: int, theta: float):
    """angle[p, i] = p * theta^(-2i/D), i < D/2 (reading A3)."""
    i = np.arange(head_dim // 2, dtype=np.float64)
    inv_freq = theta ** (-2.0 * i / head_dim)
    ang = np.asarray(positions, dtype=np.float64)[:, None] * inv_freq[None, :]
    return np.cos(ang), np.sin(ang)


def apply_rope(x: np.ndarray, cos: np.ndarray, sin: np.ndarray) -> np.ndarray:
    """Rotate-half RoPE on x [n, heads, D]: (x_i, x_{i+D/2}) ->
    (x_i cos - x_{i+D/2} sin, x_{i+D/2} cos + x_i sin) (reading A3)."""
    half = x.shape[-1] // 2
    x1, x2 = x[..., :half], x[..., half:]
    c, s = cos[:, None, :], sin[:, None, :]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


def softmax(s: np.ndarray) -> np.ndarray:
    """Max-subtracted softmax over the last axis (Eq. 2)."""
    m = np.max(s, axis=-1, keepdims=True)
    e = np.exp(s - m)
    return e / np.sum(e, axis=-1, keepdims=True)


def attention(q: np.ndarray, k: np.ndarray, v: np.ndarray,
              q_pos: np.ndarray, k_pos: np.ndarray) -> np.ndarray:
    """Eq. 2, causal: o_i = sum_{j: pos_j <= pos_i} softmax_j(q_i.k_j/sqrt(D)) v_j.

    q [S, M, D]; k, v [T, Mkv, D]; q head h reads kv head h // (M/Mkv) (A5).
    Returns o [S, M, D].
    """
    S, M, D = q.shape
    Mkv = k.shape[1]
    G = M // Mkv
    scale = 1.0 / np.sqrt(D)
    mask = np.asarray(k_pos)[None, :] <= np.asarray(q_pos)[:, None]  # [S, T]
    o = np.empty_like(q)
    for h in range(M):
        g = h // G
        s = (q[:, h, :] @ k[:, g, :].T) * scale
        s = np.where(mask, s, -np.inf)
        o[:, h, :] = softmax(s) @ v[:, g, :]
    return o


def silu(z: np.ndarray) -> np.ndarray:
    return z / (1.0 + np.exp(-z))


def greedy(logits: np.ndarray) -> int:
    """argmax, lowest index on exact ties; NaN logits are an error (A6)."""
    if np.isnan(logits).any():
        raise FloatingPointError("NaN logits")
    return int(np.argmax(logits))  # numpy returns the first maximal index


# ---------------------------------------------------------------- KV storage
@dataclass
class ContiguousKV:
    """Per-layer K/V of one sequence, [T, Mkv, D] each."""
    k: List[np.ndarray]
    v: List[np.ndarray]

    @staticmethod
    def empty(n_layers: int, n_kv: int, d: int) -> "ContiguousKV":
        z = lambda: np.zeros((0, n_kv, d))  # noqa: E731
        return ContiguousKV([z() for _ in range(n_layers)], [z() for _ in range(n_layers)])

    def append(self, layer: int, k: np.ndarray, v: np.ndarray) -> None:
        self.k[layer] = np.concatenate([self.k[layer], k], axis=0)
        self.v[layer] = np.concatenate([self.v[layer], v], axis=0)

    def get(self, layer: int):
        return self.k[layer], self.v[layer]

    @property
    def length(self) -> int:
        return self.k[0].shape[0]


@dataclass
class PagedKV:
    """C3: K/V stored through a block table into a shared pool
    pool[layer][kv] of shape [num_blocks, Mkv, 64, D]."""
    pool_k: List[np.ndarray]
    pool_v: List[np.ndarray]
    block_table: List[int] = field(default_factory=list)
    length: int = 0

    def append(self, layer: int, k: np.ndarray, v: np.ndarray, start: int) -> None:
        for j in range(k.shape[0]):
            t = start + j
            blk = self.block_table[t // BLOCK_TOKENS]
            self.pool_k[layer][blk, :, t % BLOCK_TOKENS, :] = k[j]
            self.pool_v[layer][blk, :, t % BLOCK_TOKENS, :] = v[j]

    def get(self, layer: int, n: int):
        """Gather tokens 0..n-1 in logical order."""
        ks = [self.pool_k[layer][self.block_table[t // BLOCK_TOKENS], :, t % BLOCK_TOKENS, :] for t in range(n)]
        vs = [self.pool_v[layer][self.block_table[t // BLOCK_TOKENS], :, t % BLOCK_TOKENS, :] for t in range(n)]
        return np.stack(ks), np.stack(vs)


# ---------------------------------------------------------------- the model
@dataclass
class StepOut:
    hidden: List[np.ndarray]   # residual stream before layer 0 .. after layer L-1: L+1 arrays [n, H]
    logits: np.ndarray         # [V] for the last row
    token: int


class Model:
    """fp64 decoder over bf16-exact weights (``Bf16Weights.as_f64()``)."""

    def __init__(self, shape, w64: Dict):
        self.s = shape
        self.w = w64

    # one decoder layer on rows x [n, H] at `positions`, with KV store `kv`
    def layer(self, l: int, x: np.ndarray, positions: np.ndarray, kv, paged_start: Optional[int] = None):
        s, w = self.s, self.w["layers"][l]
        M, Mkv, D = s.n_heads, s.n_kv_heads, s.head_dim
        h = rmsnorm(x, w["attn_norm"], s.rms_eps)
        q = (h @ w["wq"].T).reshape(-1, M, D)                      # Eq. 1
        k = (h @ w["wk"].T).reshape(-1, Mkv, D)
        v = (h @ w["wv"].T).reshape(-1, Mkv, D)
        cos, sin = rope_cos_sin(positions, D, s.rope_theta)
        q, k = apply_rope(q, cos, sin), apply_rope(k, cos, sin)
        if isinstance(kv, PagedKV):
            kv.append(l, k, v, paged_start)
            n_ctx = paged_start + x.shape[0]
            k_all, v_all = kv.get(l, n_ctx)
        else:
            kv.append(l, k, v)
            k_all, v_all = kv.get(l)
        k_pos = np.arange(k_all.shape[0])
        o = attention(q, k_all, v_all, positions, k_pos)             # Eq. 2
        x1 = x + o.reshape(-1, M * D) @ w["wo"].T                    # O-proj + residual
        h2 = rmsnorm(x1, w["ffn_norm"], s.rms_eps)
        a = silu(h2 @ w["w_gate"].T) * (h2 @ w["w_up"].T)             # Eq. 3 (A1)
        return x1 + a @ w["w_down"].T

    def embed(self, tokens) -> np.ndarray:
        return self.w["embed"][np.asarray(tokens, dtype=np.int64)].copy()

    def head(self, x_last: np.ndarray) -> np.ndarray:
        h = rmsnorm(x_last, self.w["final_norm"], self.s.rms_eps)
        return h @ self.w["lm_head"].T

    def forward(self, tokens, start_pos: int, kv) -> StepOut:
        """Rows `tokens` at positions start_pos.. through all layers; KV appended."""
        x = self.embed(tokens)
        positions = np.arange(start_pos, start_pos + len(tokens))
        hidden = [x]
        for l in range(self.s.n_layers):
            x = self.layer(l, x, positions, kv, paged_start=start_pos)
            hidden.append(x)
        logits = self.head(x[-1])
        return StepOut(hidden, logits, greedy(logits))

    def prefill(self, prompt, kv=None):
        """Prefill phase for one request (Fig. 2): returns (kv, StepOut)."""
        if kv is None:
            kv = ContiguousKV.empty(self.s.n_layers, self.s.n_kv_heads, self.s.head_dim)
        return kv, self.forward(prompt, 0, kv)

    def decode(self, kv, token: int, pos: int) -> StepOut:
        """One decode step: feed `token` at position `pos` (C2)."""
        return self.forward([token], pos, kv)

    def generate(self, prompt, n_tokens: int, kv=None):
        """Greedy generation of G = n_tokens tokens (prefill token + G-1 decode
        steps, reading A7). Returns (tokens, [StepOut per token])."""
        kv, out = self.prefill(prompt, kv)
        outs = [out]
        toks = [out.token]
        for k in range(1, n_tokens):
            out = self.decode(kv, toks[-1], len(prompt) + k - 1)
            outs.append(out)
            toks.append(out.token)
        return toks, outs


def forward_tp(model: Model, tokens, tp: int = 2):
    """C4: the same forward with heads [r*M/tp, (r+1)*M/tp) and FFN columns
    [r*F/tp, (r+1)*F/tp) on rank r; partial O-proj / down outputs summed over
    ranks in fp64 (two all-reduces per layer). LM head replicated.
    Returns the hidden states after each layer, [L+1][n, H]."""
    s = model.s
    M, D, F = s.n_heads, s.head_dim, s.ffn_dim
    Mkv = s.n_kv_heads
    assert M % tp == 0 and Mkv % tp == 0 and F % tp == 0
    x = model.embed(tokens)
    positions = np.arange(len(tokens))
    hidden = [x]
    for l in range(s.n_layers):
        w = model.w["layers"][l]
        h = rmsnorm(x, w["attn_norm"], s.rms_eps)
        attn_parts = []
        for r in range(tp):
            hs = slice(r * (M // tp) * D, (r + 1) * (M // tp) * D)
            ks = slice(r * (Mkv // tp) * D, (r + 1) * (Mkv // tp) * D)
            q = (h @ w["wq"][hs].T).reshape(-1, M // tp, D)
            k = (h @ w["wk"][ks].T).reshape(-1, Mkv // tp, D)
            v = (h @ w["wv"][ks].T).reshape(-1, Mkv // tp, D)
            cos, sin = rope_cos_sin(positions, D, s.rope_theta)
            q, k = apply_rope(q, cos, sin), apply_rope(k, cos, sin)
            o = attention(q, k, v, positions, positions).reshape(-1, (M // tp) * D)
            attn_parts.append(o @ w["wo"][:, hs].T)
        x = x + sum(attn_parts)                                      # all-reduce 1
        h2 = rmsnorm(x, w["ffn_norm"], s.rms_eps)
        ffn_parts = []
        for r in range(tp):
            fs = slice(r * F // tp, (r + 1) * F // tp)
            a = silu(h2 @ w["w_gate"][fs].T) * (h2 @ w["w_up"][fs].T)
            ffn_parts.append(a @ w["w_down"][:, fs].T)
        x = x + sum(ffn_parts)                                       # all-reduce 2
        hidden.append(x)
    return hidden


def top2_margin(logits: np.ndarray) -> float:
    """top1 - top2 logit (reading A20: tokens compared only where > 5e-2)."""
    part = np.partition(logits, -2)[-2:]
    return float(part[1] - part[0])
