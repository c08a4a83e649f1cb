"""Decode-GEMM configuration sweep (graph-timed): weight-streaming GB/s of the
engine's decode GEMM for r in {1, 2} weight tiles per CTA and split counts."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2504_18154_b200 import ops  # noqa: E402
from tools.gemm_decode_sweep import SHAPES, timeit  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    for name, (N, K) in SHAPES.items():
        ncopy = max(2, int(600e6 // (N * K * 2)))
        Ws = [torch.randn(N, K, device=dev).to(torch.bfloat16) for _ in range(ncopy)]
        for B in (64, 128):
            X = torch.randn(B, K, device=dev).to(torch.bfloat16)
            bn = 64 if B <= 64 else 128
            for r in (1, 3):
                for splits in (1, 2, 3, 4, 6, 8):
                    f = lambda i: ops.gemm_decode(Ws[i % ncopy], X, r, splits, bn)  # noqa: E731
                    us = timeit(f)
                    print(json.dumps(dict(op=name, B=B, r=r, splits=splits, us=round(us, 2),
                                          gbs=round(N * K * 2 / (us * 1e-6) / 1e9, 1))), flush=True)
        del Ws


if __name__ == "__main__":
    main()
