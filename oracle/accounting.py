"""ORACLE (test infrastructure only) -- FLOP / byte accounting.

* Table 2: FLOPs and memory accesses (elements) of the six
  matrix multiplications, prefill and decode columns, exactly as printed.
* KV bytes per token ("the KV cache for a single token requires 1.52 MB"):
  2 * L * Mkv * D * bytes_per_element.
* Table 3: required FuDG bandwidth = prefill token rate x KV bytes
  per token (units: GiB/s, reading A21).
* SURVEY 8(d) algorithmic work of one prefill sequence / one decode step (the
  roofline numerators bench.py reports).
"""
from __future__ import annotations

OPS = ("qkv", "qk", "av", "o", "expand", "reduce")


def table2(op: str, phase: str, B: int, S: int, H: int, M: int):
    """(flops, memory_elements) of Table 2 row `op`."""
    if phase == "prefill":
        return {
            "qkv": (6 * B * S * H * H, 6 * B * S * H + 3 * H * H),
            "qk": (2 * B * S * S * H, 2 * B * S * H + B * S * S * M),
            "av": (2 * B * S * S * H, 2 * B * S * H + B * S * S * M),
            "o": (2 * B * S * H * H, 2 * B * S * H + H * H),
            "expand": (8 * B * S * H * H, 2 * B * S * H + 4 * H * H),
            "reduce": (8 * B * S * H * H, 2 * B * S * H + 4 * H * H),
        }[op]
    if phase == "decode":
        return {
            "qkv": (6 * B * H * H, 6 * B * H + 3 * H * H),
            "qk": (2 * B * S * H, 2 * B * S * M + B * H * (S + 1)),
            "av": (2 * B * S * H, 2 * B * S * M + B * H * (S + 1)),
            "o": (2 * B * H * H, 2 * B * H + H * H),
            "expand": (8 * B * H * H, 2 * B * H + 4 * H * H),
            "reduce": (8 * B * H * H, 2 * B * H + 4 * H * H),
        }[op]
    raise ValueError(phase)


def kv_bytes_per_token(n_layers: int, n_kv_heads: int, head_dim: int, elem_bytes: int = 2) -> int:
    """K and V, every layer, one token."""
    return 2 * n_layers * n_kv_heads * head_dim * elem_bytes


def required_kv_bandwidth_gib(tokens_per_s: float, kv_bytes: int) -> float:
    """Table 3: bytes/s of KV a FuDG prefill node emits, in GiB/s."""
    return tokens_per_s * kv_bytes / 2 ** 30


def linear_params(shape) -> int:
    """P_lin: parameters of all linear layers except embed / LM head."""
    H, D, F = shape.hidden, shape.head_dim, shape.ffn_dim
    M, Mkv = shape.n_heads, shape.n_kv_heads
    per_layer = H * (M + 2 * Mkv) * D + M * D * H + 3 * H * F
    return shape.n_layers * per_layer


def prefill_flops(shape, S: int, tp: int = 1) -> int:
    """S*2*P_lin/tp + 2*L*(M/tp)*D*S(S+1) (causal QK^T + PV) + 2*H*V."""
    L, M, D = shape.n_layers, shape.n_heads, shape.head_dim
    return (S * 2 * linear_params(shape) // tp + 2 * L * (M // tp) * D * S * (S + 1)
            + 2 * shape.hidden * shape.vocab)


def decode_bytes(shape, ctx_lens, tp: int = 1) -> int:
    """weights + LM head + KV read (ctx incl. the new token) + KV write + embed rows."""
    kvtok = kv_bytes_per_token(shape.n_layers, shape.n_kv_heads // tp, shape.head_dim)
    B = len(ctx_lens)
    return (2 * linear_params(shape) // tp + 2 * shape.hidden * shape.vocab
            + sum(ctx_lens) * kvtok + B * kvtok + 2 * B * shape.hidden)


def decode_flops(shape, ctx_lens, tp: int = 1) -> int:
    L, M, D = shape.n_layers, shape.n_heads, shape.head_dim
    B = len(ctx_lens)
    return B * (2 * linear_params(shape) // tp + 2 * shape.hidden * shape.vocab) + 4 * L * (M // tp) * D * sum(ctx_lens)
