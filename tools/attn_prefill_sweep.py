"""Prefill attention microbenchmark (graph-timed): mma.sync FA2 kernel vs the
tcgen05 kernel on the Llama-3-8B head layout (M=32, Mkv=8, D=128) with a
configs[1]-like varlen batch over a paged pool."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2504_18154_b200 import ops  # noqa: E402


def timeit(fn, iters=10, rounds=3):
    """Plain CUDA-event timing (the op wrappers copy host metadata, so no graph capture);
    best of `rounds` rounds of `iters` calls."""
    fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(rounds):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(iters):
            fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / iters * 1e3)
    return best


def main():
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(0)
    M, Mkv, D = 32, 8, 128
    for lens in ([512] * 16, list(rng.integers(512, 2049, 8)), [2048] * 4, [8192]):
        nb = [(s + 63) // 64 for s in lens]
        n_blocks = sum(nb) + 8
        pool = torch.randn(n_blocks * 2 * Mkv * 64 * D, device=dev).to(torch.bfloat16)
        bt = np.zeros((len(lens), max(nb)), dtype=np.int32)
        perm = rng.permutation(n_blocks)
        k = 0
        for i, b in enumerate(nb):
            bt[i, :b] = perm[k:k + b]
            k += b
        btd = torch.from_numpy(bt).to(dev)
        cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
        q = torch.randn(int(cu[-1]), M, D, device=dev).to(torch.bfloat16)
        flop = sum(2 * M * D * s * (s + 1) for s in lens)
        t_mma = timeit(lambda: ops.attention_prefill(q, pool, n_blocks, M, Mkv, D, cu, btd))
        t_tc = timeit(lambda: ops.attention_prefill_tc(q, pool, n_blocks, M, Mkv, cu, btd))
        print(json.dumps(dict(tokens=int(cu[-1]), n_seq=len(lens), mma_us=round(t_mma, 1),
                              mma_tflops=round(flop / t_mma / 1e6, 1), tc_us=round(t_tc, 1),
                              tc_tflops=round(flop / t_tc / 1e6, 1))), flush=True)


if __name__ == "__main__":
    main()
