"""Runs a few decode-shaped GEMMs (for ncu captures): GU (28672x4096) unsplit and
QKV (6144x4096) split 3, B=128."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2504_18154_b200 import ops  # noqa: E402

dev = torch.device("cuda", 0)
X = torch.randn(128, 4096, device=dev).to(torch.bfloat16)
Wgu = torch.randn(28672, 4096, device=dev).to(torch.bfloat16)
Wqkv = torch.randn(6144, 4096, device=dev).to(torch.bfloat16)
for _ in range(2):
    ops.gemm_decode(Wgu, X, 1, 1, 128)
    ops.gemm_decode(Wqkv, X, 1, 3, 128)
torch.cuda.synchronize()
print("ok")
