"""KV migration between instances (N1 / K11): a running request moved mid-decode
with its paged KV continues bit-exactly -- the tokens after the move equal the
tokens of the same request decoded without moving (rows are independent in
every kernel, so batch composition cannot change a request's result). Same GPU
and, when 2 GPUs are visible, across NVLink."""
import numpy as np
import pytest
import torch

from synthetic.shapes import get_shape
from synthetic.traces import make_trace
from synthetic.weights import make_weights

pytestmark = pytest.mark.gpu


def _pair(dev_b):
    from paper_2504_18154_b200.instance import Instance, device_weights_from_host
    shape = get_shape("tiny-gqa")
    w = make_weights(shape, seed=0)
    a = Instance(shape, device_weights_from_host(w, "cuda:0"), 64, 0, token_budget=2048, max_batch=32,
                 max_positions=2048)
    b = Instance(shape, device_weights_from_host(w, f"cuda:{dev_b}"), 64, dev_b, token_budget=2048, max_batch=32,
                 max_positions=2048)
    return shape, a, b


@pytest.mark.parametrize("dev_b", [0, 1])
def test_migrate_mid_decode_is_bitexact(dev_b):
    if dev_b >= torch.cuda.device_count():
        pytest.skip("cross-GPU migration needs 2 GPUs")
    shape, a, b = _pair(dev_b)
    reqs = make_trace("tiny", 4, seed=4, vocab=shape.vocab)
    ids = [r.req_id for r in reqs]
    # reference: everything on A, 20 tokens
    a.prefill([(100 + r.req_id, r.prompt, 20) for r in reqs])
    ref, _ = a.decode([100 + i for i in ids], 19)
    a.release([100 + i for i in ids])
    # migrated: 7 decode steps on A, move requests 1 and 3 to B, continue both
    a.prefill([(r.req_id, r.prompt, 20) for r in reqs])
    t1, _ = a.decode(ids, 7)
    blocks_before = a.status()[0]["blocks_used"]
    moved = [a.migrate_to(b, rid) for rid in (1, 3)]
    assert all(m["n_generated"] == 8 for m in moved)
    assert a.status()[0]["blocks_used"] == blocks_before - sum(m["n_blocks"] for m in moved)
    ta, _ = a.decode([0, 2], 12)
    tb, _ = b.decode([1, 3], 12)
    got = np.zeros_like(ref)
    got[:, :7] = t1
    got[[0, 2], 7:] = ta
    got[[1, 3], 7:] = tb
    assert np.array_equal(got, ref)
    a.close()
    b.close()
