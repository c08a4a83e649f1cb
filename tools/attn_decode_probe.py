"""Decode attention kernel alone (TMA path, 8B geometry M32 Mkv8 D128, one layer pool):
device time and KV GB/s for several (B, context) pairs with the same KV bytes -- how
much per-CTA start-up / wave structure costs. Pools are several GB (beyond L2)."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(B, ctx, M=32, Mkv=8, D=128, reps=10, sk=False):
    from paper_2504_18154_b200 import ops
    nb = (ctx + 63) // 64
    n_blocks = B * nb + 8
    pool = torch.randn(n_blocks, 2, Mkv, 64, D, device="cuda").to(torch.bfloat16)
    perm = torch.randperm(n_blocks, device="cuda", dtype=torch.int64)[: B * nb].to(torch.int32)
    bt = perm.view(B, nb).contiguous()
    q = torch.randn(B, M, D, device="cuda").to(torch.bfloat16)
    cl = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
    ctx_list = [ctx] * B

    def call():
        if sk:
            ops.attention_decode_sk(q, pool, M, Mkv, D, ctx_list, bt)
        else:
            ops.attention_decode(q, pool, M, Mkv, D, cl, bt, 1, nb, use_tma=True)
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        a.record()
        call()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    us = sorted(ts)[len(ts) // 2]
    byts = B * ctx * Mkv * D * 2 * 2
    print(json.dumps({"sk": sk, "B": B, "ctx": ctx, "ctas": B * Mkv, "us": round(us, 2), "gbs": round(byts / us / 1e3, 1)}),
          flush=True)


if __name__ == "__main__":
    for B, ctx in [(128, 1300), (64, 2600), (128, 2600), (256, 650)]:
        run(B, ctx)
        run(B, ctx, sk=True)
