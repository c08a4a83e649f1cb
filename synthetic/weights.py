"""Seeded random-init weights, stored as bf16 bit patterns (uint16).

Recipe (SURVEY.md 8(d) "Weight init"): E ~ N(0,1); W ~ N(0, 1/fan_in);
gamma ~ 1 + U(-0.1, 0.1); W_lm ~ N(0, (2/sqrt(H))^2). Every tensor is drawn in
fp32 from its own numpy PCG64 stream keyed by (seed, layer, tensor) and rounded
to bf16 with round-to-nearest-even, so the oracle and the CUDA path use the
exact same weight values (weight quantisation is not part of
the error budget).

Layout: every matrix is [out, in] row-major (the C ABI's layout).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List

import numpy as np

from .shapes import ModelShape

LAYER_TENSORS = ("attn_norm", "wq", "wk", "wv", "wo",
                 "ffn_norm", "w_gate", "w_up", "w_down")


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round fp32 -> bf16 (round to nearest, ties to even); returns uint16 bits."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    rounding = np.uint32(0x7FFF) + ((b >> np.uint32(16)) & np.uint32(1))
    return ((b + rounding) >> np.uint32(16)).astype(np.uint16)


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def layer_shapes(s: ModelShape) -> Dict[str, tuple]:
    H, D, F = s.hidden, s.head_dim, s.ffn_dim
    return {
        "attn_norm": (H,),
        "wq": (s.n_heads * D, H),
        "wk": (s.n_kv_heads * D, H),
        "wv": (s.n_kv_heads * D, H),
        "wo": (H, s.n_heads * D),
        "ffn_norm": (H,),
        "w_gate": (F, H),
        "w_up": (F, H),
        "w_down": (H, F),
    }


def _rng(seed: int, layer: int, tensor: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, layer + 1, tensor])))


def _draw(name: str, shape: tuple, rng: np.random.Generator, hidden: int) -> np.ndarray:
    if name.endswith("norm"):
        return (1.0 + rng.uniform(-0.1, 0.1, size=shape)).astype(np.float32)
    if name == "embed":
        return rng.standard_normal(shape, dtype=np.float32)
    if name == "lm_head":
        return rng.standard_normal(shape, dtype=np.float32) * np.float32(2.0 / np.sqrt(hidden))
    fan_in = shape[1]
    return rng.standard_normal(shape, dtype=np.float32) * np.float32(1.0 / np.sqrt(fan_in))


@dataclass
class Bf16Weights:
    """Host copy of a model's weights as bf16 bit patterns."""
    shape: ModelShape
    embed: np.ndarray            # uint16 [V, H]
    lm_head: np.ndarray          # uint16 [V, H]
    final_norm: np.ndarray       # uint16 [H]
    layers: List[Dict[str, np.ndarray]] = field(default_factory=list)

    def as_f64(self):
        """fp64 copies (exact: every bf16 value is representable)."""
        cv = lambda a: bf16_bits_to_f32(a).astype(np.float64)  # noqa: E731
        return {
            "embed": cv(self.embed),
            "lm_head": cv(self.lm_head),
            "final_norm": cv(self.final_norm),
            "layers": [{k: cv(v) for k, v in l.items()} for l in self.layers],
        }


def make_weights(shape: ModelShape, seed: int = 0) -> Bf16Weights:
    H, V = shape.hidden, shape.vocab
    embed = f32_to_bf16_bits(_draw("embed", (V, H), _rng(seed, -1, 0), H))
    lm_head = f32_to_bf16_bits(_draw("lm_head", (V, H), _rng(seed, -1, 1), H))
    final_norm = f32_to_bf16_bits(_draw("final_norm", (H,), _rng(seed, -1, 2), H))
    layers = []
    shp = layer_shapes(shape)
    for l in range(shape.n_layers):
        layers.append({name: f32_to_bf16_bits(_draw(name, shp[name], _rng(seed, l, i), H))
                       for i, name in enumerate(LAYER_TENSORS)})
    return Bf16Weights(shape, embed, lm_head, final_norm, layers)
