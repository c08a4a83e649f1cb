"""Per-step timeline of one decode-chain launch (layer 1) from %globaltimer marks.
  ECOSERVE_CHAIN_TRACE=/path python tools/chain_trace.py [shape] [batch] [prompt]
then prints, per chain step: when the producer passed the step's barrier (median / max
over CTAs), the first accumulator, and the CTAs' arrivals (min / max)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(shape_name, batch, prompt, path):
    import torch
    from paper_2504_18154_b200 import build as B
    B.build()
    from paper_2504_18154_b200.instance import Instance, random_device_weights
    from synthetic.shapes import get_shape
    shape = get_shape(shape_name)
    dev = torch.device("cuda", 0)
    w = random_device_weights(shape, seed=1, device=dev)
    blocks = batch * ((prompt + 64) // 64 + 2) + 64
    inst = Instance(shape, w, blocks, 0, token_budget=16384, max_batch=max(256, batch), max_positions=prompt + 512,
                    free_raw_after_create=True)
    rng = np.random.default_rng(0)
    for i in range(0, batch, 16):
        inst.prefill([(j, rng.integers(0, shape.vocab, prompt).astype(np.int32), 512) for j in range(i, i + 16)])
    if os.path.exists(path):
        os.remove(path)
    inst.decode(list(range(batch)), 3)
    inst.close()


def analyse(path):
    blocks, cur = [], None
    for line in open(path):
        if line.startswith("#"):
            cur = []
            blocks.append(cur)
            continue
        cur.append([int(v) for v in line.split()])
    d = np.array(blocks[-1])
    n_steps = d[:, 1].max() + 1
    print(f"{'step':>4} {'prod pass med/max us':>22} {'first acc med':>14} {'arrive min/max us':>20}")
    for si in range(n_steps):
        def sel(k):
            m = (d[:, 1] == si) & (d[:, 2] == k)
            return d[m, 3] / 1e3
        p, a, r = sel(0), sel(1), sel(2)
        f = lambda x, fn: f"{fn(x):8.1f}" if len(x) else "       -"
        print(f"{si:>4} {f(p, np.median)} {f(p, np.max)}   {f(a, np.median)}   {f(r, np.min)} {f(r, np.max)}")


if __name__ == "__main__":
    path = os.environ.get("ECOSERVE_CHAIN_TRACE", "/tmp/chain_trace.txt")
    if len(sys.argv) > 1 and sys.argv[1] == "--analyse":
        analyse(sys.argv[2] if len(sys.argv) > 2 else path)
    else:
        run(sys.argv[1] if len(sys.argv) > 1 else "8b", int(sys.argv[2]) if len(sys.argv) > 2 else 128,
            int(sys.argv[3]) if len(sys.argv) > 3 else 1024, path)
        analyse(path)
