"""Prefill GEMM microbenchmark (graph-timed): TFLOP/s of the 1-CTA 128x256 and the
CTA-pair 256x256 tcgen05 kernels on the Llama-3-8B prefill projection shapes."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2504_18154_b200 import ops  # noqa: E402

SHAPES = {"qkv": (6144, 4096), "o": (4096, 4096), "gu": (28672, 4096), "down": (4096, 14336)}


def timeit(fn, iters=10):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(iters):
            fn()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3


def main():
    dev = torch.device("cuda", 0)
    for T in (4096, 10240, 16384):
        for name, (N, K) in SHAPES.items():
            A = torch.randn(T, K, device=dev).to(torch.bfloat16)
            W = torch.randn(N, K, device=dev).to(torch.bfloat16)
            for bn in (256, 2):
                us = timeit(lambda: ops.gemm(A, W, torch.bfloat16, bn))
                print(json.dumps(dict(T=T, op=name, bn=bn, us=round(us, 1), tflops=round(2 * T * N * K / us / 1e6, 1))),
                      flush=True)


if __name__ == "__main__":
    main()
