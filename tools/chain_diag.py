"""Per-layer decode hidden states vs the oracle, one decode step at a time
(teacher-forced on the GPU's own tokens): locates where a decode path diverges.
  python tools/chain_diag.py [shape] [steps]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import transformer as T  # noqa: E402
from synthetic.shapes import get_shape  # noqa: E402
from synthetic.traces import make_trace  # noqa: E402
from synthetic.weights import make_weights  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "tiny"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    from paper_2504_18154_b200 import build as B
    B.build()
    from paper_2504_18154_b200.instance import Instance, device_weights_from_host
    shape = get_shape(name)
    w = make_weights(shape, seed=0)
    inst = Instance(shape, device_weights_from_host(w, "cuda:0"), 64, 0, token_budget=4096, max_batch=64,
                    max_positions=4096, debug_hidden=True)
    model = T.Model(shape, w.as_f64())
    reqs = make_trace("tiny", 8, seed=1, vocab=shape.vocab)
    first = inst.prefill([(r.req_id, r.prompt, r.output_len) for r in reqs])
    state = {}
    for i, r in enumerate(reqs):
        kv, out = model.prefill(list(r.prompt))
        state[r.req_id] = [kv, int(first[i]), r.prompt_len]
    ids = [r.req_id for r in reqs]
    worst_all = 0.0
    for s in range(steps):
        toks, _ = inst.decode(ids, 1)
        worst = np.zeros(shape.n_layers + 1)
        for i, rid in enumerate(ids):
            kv, tok, pos = state[rid]
            out = model.decode(kv, tok, pos)
            for l in range(shape.n_layers + 1):
                got = inst.hidden(rid, l, 1)[0]
                ref = out.hidden[l].reshape(-1)
                worst[l] = max(worst[l], float(np.max(np.abs(got - ref)) / np.max(np.abs(ref))))
            state[rid] = [kv, int(toks[i, 0]), pos + 1]
        print(f"step {s}: worst per-layer rel err {np.array2string(worst, precision=4)}", flush=True)
        worst_all = max(worst_all, float(worst.max()))
    inst.close()
    print(f"WORST {worst_all:.6f}", flush=True)
    return worst_all


if __name__ == "__main__":
    tol = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-2
    sys.exit(0 if main() <= tol else 1)
