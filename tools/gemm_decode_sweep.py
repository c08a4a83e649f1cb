"""Microbenchmark of the decode-shaped (swap-AB, split-K) GEMM on the GPU:
achieved weight-streaming GB/s per (N, K, B, splits, path) for the Llama-3-8B
decode projections. Timed with CUDA events over repeated launches, inputs far
larger than L2 cycled between iterations."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2504_18154_b200 import ops  # noqa: E402

SHAPES = {"qkv": (6144, 4096), "o": (4096, 4096), "gu": (28672, 4096), "down": (4096, 14336)}


def timeit(fn, iters=20):
    """Capture `iters` calls in a CUDA graph and time its replay (no host overhead)."""
    for _ in range(2):
        fn(0)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(iters):
            fn(i)
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3  # us


def main():
    res = []
    dev = torch.device("cuda", 0)
    for name, (N, K) in SHAPES.items():
        # several weight copies so consecutive launches stream from HBM, not L2
        ncopy = max(2, int(600e6 // (N * K * 2)))
        Ws = [torch.randn(N, K, device=dev).to(torch.bfloat16) for _ in range(ncopy)]
        for B in (64, 128, 256):
            X = torch.randn(B, K, device=dev).to(torch.bfloat16)
            bn = 64 if B <= 64 else 128 if B <= 128 else 256
            for splits in (1, 2, 3, 4, 6, 8):
                for path in ("reduce_kernel", "inkernel") if splits == 1 else ("reduce_kernel",):
                    if path == "inkernel":
                        f = lambda i: ops.gemm_swap_bf16(Ws[i % ncopy], X, splits, bn)  # noqa: E731
                    else:
                        f = lambda i: ops.gemm_swap(Ws[i % ncopy], X, splits, bn)  # noqa: E731
                    us = timeit(f)
                    gbs = N * K * 2 / (us * 1e-6) / 1e9
                    res.append(dict(op=name, N=N, K=K, B=B, splits=splits, path=path, us=round(us, 2),
                                    gbs=round(gbs, 1)))
                    print(json.dumps(res[-1]), flush=True)
        del Ws


if __name__ == "__main__":
    main()
