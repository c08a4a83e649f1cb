"""KV migration between two instances on two B200s (mitosis
contraction / rebalancing moves running requests with their paged KV; the paper
reports migration well under 100 ms). Llama-3-8B shape, requests of
1k-8k tokens prefilled on GPU 0 and moved to GPU 1 (export into a staging buffer on
the destination over NVLink, import, release); wall time of Instance.migrate_to.

  python tools/migrate_bench.py
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_2504_18154_b200 import build as B
    B.build(verbose=False)
    from paper_2504_18154_b200.instance import Instance, random_device_weights
    from synthetic.shapes import get_shape
    if torch.cuda.device_count() < 2:
        print(json.dumps({"skipped": "needs 2 GPUs"}))
        return
    shape = get_shape("8b")
    insts = []
    for g in range(2):
        torch.cuda.set_device(g)
        w = random_device_weights(shape, seed=5, device=torch.device("cuda", g))
        insts.append(Instance(shape, w, 2000, g, token_budget=16384, max_batch=64, max_positions=9216,
                              free_raw_after_create=True))
    a, b = insts
    rng = np.random.default_rng(0)
    rows = []
    rid = 1
    for S in (1024, 4096, 8192):
        for rep in range(3):
            a.prefill([(rid, rng.integers(0, shape.vocab, S).astype(np.int32), 64)])
            a.decode([rid], 2)
            torch.cuda.synchronize(0)
            torch.cuda.synchronize(1)
            t0 = time.perf_counter()
            info = a.migrate_to(b, rid)
            dt = time.perf_counter() - t0
            toks, _ = b.decode([rid], 2)  # the request continues on the destination
            assert (toks >= 0).all()
            b.release([rid])
            if rep > 0:
                rows.append({"prompt": S, "blocks": info["n_blocks"], "mb": round(info["bytes"] / 2 ** 20, 1),
                             "ms": round(dt * 1e3, 3), "gb_s": round(info["bytes"] / dt / 1e9, 1)})
            rid += 1
    for r in rows:
        print(json.dumps(r), flush=True)
    for i in insts:
        i.close()


if __name__ == "__main__":
    main()
