"""End-to-end parity of the PaDG instance (prefill phase + decode phase through
the C ABI) against the fp64 oracle, BASELINE.json configs[0] (tiny decoder, 8
requests, prompts 32-128, 16 output tokens = 1 prefill + 15 decode steps).

Bars (north star; readings A19, A20 in DESIGN.md):
* residual stream after every layer: max|h_gpu - h_ref| / max|h_ref| <= 1e-2;
* greedy tokens equal wherever the oracle's top1-top2 logit margin > 5e-2
  (a sequence is compared up to its first legitimate divergence, i.e. a step
  whose oracle margin is <= 5e-2).
"""
import numpy as np
import pytest
import torch

from oracle import transformer as T
from synthetic.shapes import get_shape
from synthetic.traces import make_trace
from synthetic.weights import make_weights

pytestmark = pytest.mark.gpu

HID_TOL = 1e-2
MARGIN = 5e-2


def build(name, n_blocks=64, debug=True, token_budget=4096):
    from paper_2504_18154_b200.instance import Instance, device_weights_from_host
    shape = get_shape(name)
    w = make_weights(shape, seed=0)
    inst = Instance(shape, device_weights_from_host(w, "cuda:0"), n_blocks, 0, token_budget=token_budget,
                    max_batch=64, max_positions=4096, debug_hidden=debug)
    return shape, w, inst


def rel(a, b):
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


@pytest.mark.parametrize("name", ["tiny", "tiny-gqa", "tiny-d128"])
def test_tiny_prefill_then_decode(name):
    shape, w, inst = build(name)
    model = T.Model(shape, w.as_f64())
    reqs = make_trace("tiny", 8, seed=1, vocab=shape.vocab)
    first = inst.prefill([(r.req_id, r.prompt, r.output_len) for r in reqs])
    ref = {}
    for r in reqs:
        kv, out = model.prefill(list(r.prompt))
        ref[r.req_id] = (kv, out)
        for l in range(shape.n_layers + 1):
            got = inst.hidden(r.req_id, l, r.prompt_len)
            assert rel(got, out.hidden[l]) <= HID_TOL, (r.req_id, l, rel(got, out.hidden[l]))
    # first tokens
    live = {}
    for i, r in enumerate(reqs):
        kv, out = ref[r.req_id]
        if first[i] != out.token:
            assert T.top2_margin(out.logits) <= MARGIN
        else:
            live[r.req_id] = (kv, out.token)
    # decode: 15 steps, compared step by step until a legitimate divergence
    steps = reqs[0].output_len - 1
    toks, nf = inst.decode([r.req_id for r in reqs], steps)
    assert nf == len(reqs)
    checked = 0
    for i, r in enumerate(reqs):
        if r.req_id not in live:
            continue
        kv, tok = live[r.req_id]
        for s in range(steps):
            out = model.decode(kv, tok, r.prompt_len + s)
            if toks[i, s] != out.token:
                assert T.top2_margin(out.logits) <= MARGIN, (r.req_id, s)
                break
            checked += 1
            tok = out.token
            if s == steps - 1:   # last step: hidden states of the decode row
                for l in range(shape.n_layers + 1):
                    got = inst.hidden(r.req_id, l, 1)
                    assert rel(got, out.hidden[l][-1:]) <= HID_TOL, (r.req_id, l)
    # free-running greedy sequences stop being comparable at the first legitimate flip of a
    # near tie (top-2 margin <= 5e-2: ~10 % of steps at this logit scale), so how many steps
    # get compared depends on rounding order (e.g. where the prefill RMSNorm is applied);
    # the per-layer hidden-state bar above is the precise check
    assert checked >= 0.6 * len(reqs) * steps
    st, rs = inst.status()
    assert st["alive"] and st["n_requests"] == 8 and all(x["finished"] for x in rs)
    inst.release([r.req_id for r in reqs])
    st, _ = inst.status()
    assert st["blocks_used"] == 0
    inst.close()


@pytest.mark.parametrize("name", ["tiny", "tiny-gqa", "tiny-d128"])
def test_tiny_teacher_forced_decode(name):
    """Reading A20 as written: the oracle's greedy sequence is teacher-forced on the GPU
    (ecoserve_debug_force_token before every decode step), so every one of the 8 x 15
    steps is comparable: the GPU's argmax must equal the oracle's wherever the oracle's
    top-2 margin exceeds 5e-2, and the decode row's residual stream after every layer is
    within the A19 bar at every step (the KV it attends over was written by the GPU's own
    earlier steps on the same forced ids)."""
    shape, w, inst = build(name)
    model = T.Model(shape, w.as_f64())
    reqs = make_trace("tiny", 8, seed=1, vocab=shape.vocab)
    first = inst.prefill([(r.req_id, r.prompt, r.output_len) for r in reqs])
    state = {}
    for i, r in enumerate(reqs):
        kv, out = model.prefill(list(r.prompt))
        state[r.req_id] = [kv, out.token]
        if first[i] != out.token:
            assert T.top2_margin(out.logits) <= MARGIN, (r.req_id, T.top2_margin(out.logits))
    steps = reqs[0].output_len - 1
    ids = [r.req_id for r in reqs]
    checked = total = 0
    worst = 0.0
    for s in range(steps):
        for r in reqs:
            inst.force_token(r.req_id, state[r.req_id][1])
        toks, _ = inst.decode(ids, 1)
        for i, r in enumerate(reqs):
            kv, tok = state[r.req_id]
            out = model.decode(kv, tok, r.prompt_len + s)
            total += 1
            if T.top2_margin(out.logits) > MARGIN:
                assert toks[i, 0] == out.token, (r.req_id, s, int(toks[i, 0]), out.token)
                checked += 1
            for l in range(shape.n_layers + 1):
                e = rel(inst.hidden(r.req_id, l, 1), out.hidden[l][-1:])
                worst = max(worst, e)
                assert e <= HID_TOL, (r.req_id, s, l, e)
            state[r.req_id][1] = out.token
    print(f"{name}: {checked}/{total} steps with margin > {MARGIN} compared, worst hidden rel {worst:.2e}")
    assert checked >= 0.8 * total    # the weight recipe gives ~88-92 %
    with pytest.raises(Exception):
        inst.force_token(reqs[0].req_id, shape.vocab)   # out of range
    inst.release(ids)
    inst.close()


def test_kv_exhausted_is_all_or_nothing():
    shape, w, inst = build("tiny", n_blocks=4, debug=False)
    rng = np.random.default_rng(0)
    from paper_2504_18154_b200._lib import EcoError
    with pytest.raises(EcoError) as e:
        inst.prefill([(1, rng.integers(0, 1024, 200).astype(np.int32), 4),
                      (2, rng.integers(0, 1024, 100).astype(np.int32), 4)])   # needs 4 + 2 blocks
    assert e.value.status == 2
    st, _ = inst.status()
    assert st["blocks_used"] == 0 and st["n_requests"] == 0
    first = inst.prefill([(3, rng.integers(0, 1024, 256).astype(np.int32), 3)])   # exactly 4 blocks
    with pytest.raises(EcoError) as e:   # position 256 needs a 5th block
        inst.decode([3], 1)
    assert e.value.status == 2
    with pytest.raises(EcoError) as e:
        inst.prefill([(3, rng.integers(0, 1024, 10).astype(np.int32), 3)])   # duplicate id
    assert e.value.status == 3
    inst.close()


def test_batching_is_invisible():
    """The same requests prefilled together, split across token-budget batches,
    or one by one give identical tokens (rows are independent)."""
    shape, w, inst = build("tiny", n_blocks=128, debug=False, token_budget=256)
    reqs = make_trace("tiny", 6, seed=5, vocab=shape.vocab)
    a = inst.prefill([(r.req_id, r.prompt, 8) for r in reqs])           # several 256-token batches
    b = [inst.prefill([(100 + r.req_id, r.prompt, 8)])[0] for r in reqs]
    assert list(a) == list(b)
    ta, _ = inst.decode([r.req_id for r in reqs], 7)
    tb, _ = inst.decode([100 + r.req_id for r in reqs], 7)
    assert (ta == tb).all()
    inst.close()
