"""Model shapes (Table 1 notation: L, H, M, D; plus Mkv, F, V).

Shapes follow SURVEY.md section 8 "Shapes": the tiny decoder of BASELINE.json
configs[0], the Llama-3-8B shape (configs[1]), the CodeLlama-34B shape (a paper
model; configs[2]) and the Llama-2-70B shape per TP=2 rank (configs[3]).
"""
from __future__ import annotations

from dataclasses import dataclass, replace


@dataclass(frozen=True)
class ModelShape:
    name: str
    n_layers: int      # L
    hidden: int        # H
    n_heads: int       # M
    n_kv_heads: int    # Mkv (GQA)
    head_dim: int      # D
    ffn_dim: int       # F (SwiGLU width, reading A1)
    vocab: int         # V
    rope_theta: float  # reading A3
    rms_eps: float = 1e-5  # reading A4
    tp_size: int = 1

    @property
    def group(self) -> int:
        return self.n_heads // self.n_kv_heads

    @property
    def qkv_dim(self) -> int:
        return (self.n_heads + 2 * self.n_kv_heads) * self.head_dim

    def with_layers(self, n_layers: int) -> "ModelShape":
        return replace(self, n_layers=n_layers, name=f"{self.name}-L{n_layers}")


SHAPES = {
    "tiny": ModelShape("tiny", 2, 256, 8, 8, 32, 768, 1024, 1e4),
    "tiny-gqa": ModelShape("tiny-gqa", 2, 256, 8, 2, 32, 768, 1024, 1e4),
    # D=128 variant of the tiny decoder: exercises the production head_dim
    "tiny-d128": ModelShape("tiny-d128", 2, 512, 4, 2, 128, 1024, 2048, 1e4),
    "8b": ModelShape("8b", 32, 4096, 32, 8, 128, 14336, 128256, 5e5),
    "34b": ModelShape("34b", 48, 8192, 64, 8, 128, 22016, 32000, 1e6),
    "70b": ModelShape("70b", 80, 8192, 64, 8, 128, 28672, 32000, 1e4),
}


def get_shape(name: str) -> ModelShape:
    """`name` or `name-L<k>` (the same shape cut to k layers)."""
    if name in SHAPES:
        return SHAPES[name]
    base, _, layers = name.rpartition("-L")
    if base in SHAPES and layers.isdigit():
        return SHAPES[base].with_layers(int(layers))
    raise KeyError(f"unknown model shape {name!r}; known: {sorted(SHAPES)}")
