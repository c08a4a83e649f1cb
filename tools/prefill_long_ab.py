"""Prefill-phase time of long prompts (configs[4]-like: U{6144..8192}) on one instance:
device ms per prefill phase from the instance's phase events; run once per environment
(e.g. ECOSERVE_ATTN_T128=0 vs unset) in separate processes.
  python tools/prefill_long_ab.py [shape] [n_req]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    from paper_2504_18154_b200.instance import Instance, random_device_weights
    from synthetic.shapes import get_shape
    name = sys.argv[1] if len(sys.argv) > 1 else "8b"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    shape = get_shape(name)
    w = random_device_weights(shape, seed=1000, device=torch.device("cuda", 0))
    inst = Instance(shape, w, 2000, 0, token_budget=16384, max_batch=64, max_positions=9000,
                    free_raw_after_create=True)
    rng = np.random.default_rng(5)
    lens = [int(x) for x in rng.integers(6144, 8193, n)]
    res = []
    for rep in range(4):
        ids = [1000 * rep + i for i in range(n)]
        inst.timing(reset=True)
        inst.prefill([(i, rng.integers(0, shape.vocab, L).astype(np.int32), 2) for i, L in zip(ids, lens)])
        t = inst.timing(reset=True)
        inst.release(ids)
        if rep > 0:
            res.append(t["prefill_ms"])
    print(json.dumps({"shape": name, "lens": lens, "env": {k: v for k, v in os.environ.items() if k.startswith("ECOSERVE_")},
                      "prefill_ms": round(min(res), 3), "tok_s": round(sum(lens) / min(res) * 1e3, 1),
                      "all": [round(x, 3) for x in res]}), flush=True)
    inst.close()


if __name__ == "__main__":
    main()
