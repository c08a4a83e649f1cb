"""Hybrid batching (chunked prefill + decode in one forward pass, SURVEY 8(f) N3 --
the Sarathi-style NoDG baseline on these kernels) against the fp64 oracle.

A long prompt is prefilled in three chunks while other requests join and decode in
the same forward passes. Bars as in test_gpu_instance (readings A19/A20): the
residual stream of every chunk's rows after every layer is within 1e-2 of the
oracle's full (unchunked) prefill at the same positions, and greedy tokens match the
oracle wherever its top-2 margin exceeds 5e-2."""
import numpy as np
import pytest

from oracle import transformer as T
from synthetic.shapes import get_shape
from synthetic.traces import random_prompts
from synthetic.weights import make_weights

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


def tokens_match(model, prompt, got, margin=5e-2):
    toks, outs = model.generate(list(prompt), len(got))
    for k, g in enumerate(got):
        if g != toks[k]:
            assert T.top2_margin(outs[k].logits) <= margin, (k, g, toks[k])
            return k
    return len(got)


@pytest.mark.parametrize("name", ["tiny-d128", "tiny-gqa"])
def test_chunked_prefill_with_concurrent_decode(name):
    from paper_2504_18154_b200.instance import Instance, device_weights_from_host
    shape = get_shape(name)
    w = make_weights(shape, seed=0)
    model = T.Model(shape, w.as_f64())
    inst = Instance(shape, device_weights_from_host(w, "cuda:0"), 256, 0, token_budget=2048, max_batch=64,
                    max_positions=2048, debug_hidden=True)
    pa, pb, pc = random_prompts(11, [300, 150, 90], shape.vocab)
    G = 6
    gen = {1: [], 2: [], 3: []}
    # step 1: chunks of A and B
    ct, dt = inst.hybrid_step([(1, pa, G, 128), (2, pb, G, 100)], [])
    assert list(ct) == [-1, -1] and len(dt) == 0
    # step 2: A continues, B completes its prompt
    ct, dt = inst.hybrid_step([(1, pa, G, 128), (2, pb, G, 50)], [])
    assert ct[0] == -1 and ct[1] >= 0
    gen[2].append(int(ct[1]))
    # step 3: A's last chunk (compare its rows), C in one chunk, B decodes
    ct, dt = inst.hybrid_step([(1, pa, G, 44), (3, pc, G, 90)], [2])
    gen[1].append(int(ct[0]))
    gen[3].append(int(ct[1]))
    gen[2].append(int(dt[0]))
    _, out_a = model.prefill(list(pa))
    for l in range(shape.n_layers + 1):
        got = inst.hidden(1, l, 44)
        assert rel(got, out_a.hidden[l][256:300]) <= 1e-2, l
    # decode-only hybrid steps
    for _ in range(G - 1):
        live = [r for r in (1, 2, 3) if len(gen[r]) < G]
        if not live:
            break
        _, dt = inst.hybrid_step([], live)
        for r, t in zip(live, dt):
            gen[r].append(int(t))
    for rid, p in ((1, pa), (2, pb), (3, pc)):
        assert tokens_match(model, p, gen[rid][:G]) >= 2, rid
    # state errors: a chunk for a prefilled request, a decode of an unprefilled one
    from paper_2504_18154_b200 import _lib as L
    with pytest.raises(L.EcoError):
        inst.hybrid_step([(1, pa, G, 1)], [])
    inst.hybrid_step([(9, pa, G, 64)], [])
    with pytest.raises(L.EcoError):
        inst.hybrid_step([], [9])
    inst.release([1, 2, 3, 9])
    assert inst.status()[0]["blocks_used"] == 0
    inst.close()
