"""Live PaDG serving loop (paper_2504_18154_b200/serve.py) on CPU with fake
instances whose phase calls sleep for a scaled cost-model duration: checks the
threading, status plumbing, temporal disaggregation and rolling activation
logic that drives the real GPU instances (the GPU variant is in
test_gpu_serve.py)."""
import time

import numpy as np
import pytest

from synthetic.traces import make_trace

SEC = 1_000_000_000


class FakeInstance:
    """prefill/decode/release with the instance API; durations from a cost model."""

    def __init__(self, num_blocks=100000, scale=0.02):
        self.num_blocks = num_blocks
        self.scale = scale
        self.gen = {}
        self.calls = []

    def prefill(self, reqs):
        dur = sum(2e-3 + 14.3e-6 * len(p) for _, p, _ in reqs)
        time.sleep(dur * self.scale)
        self.calls.append(("prefill", len(reqs)))
        out = []
        for rid, p, g in reqs:
            assert rid not in self.gen
            self.gen[rid] = [1, g]
            out.append(int(rid % 997))
        return np.array(out, dtype=np.int32)

    def decode(self, ids, steps):
        time.sleep((3.3e-3 + 1e-6 * len(ids)) * steps * self.scale)
        self.calls.append(("decode", len(ids)))
        toks = np.full((len(ids), steps), -1, dtype=np.int32)
        for i, rid in enumerate(ids):
            for s in range(steps):
                n, g = self.gen[rid]
                if n < g:
                    self.gen[rid][0] += 1
                    toks[i, s] = (rid + n) % 997
        return toks, 0

    def hybrid_step(self, chunks, decode_ids):
        toks = sum(c[3] for c in chunks) + len(decode_ids)
        time.sleep((2e-3 + 14.3e-6 * toks) * self.scale)
        self.calls.append(("hybrid", len(chunks), len(decode_ids), toks))
        if not hasattr(self, "pre"):
            self.pre = {}
        ct = []
        for rid, p, g, take in chunks:
            st = self.pre.setdefault(rid, [0, len(p)])
            assert rid not in self.gen and 0 < take <= st[1] - st[0]
            st[0] += take
            if st[0] == st[1]:
                self.gen[rid] = [1, g]
                ct.append(int(rid % 997))
            else:
                ct.append(-1)
        dt = []
        for rid in decode_ids:
            n, g = self.gen[rid]
            assert n < g
            self.gen[rid][0] += 1
            dt.append((rid + n) % 997)
        return np.array(ct, dtype=np.int32), np.array(dt, dtype=np.int32)

    def release(self, ids):
        for rid in ids:
            del self.gen[rid]
            getattr(self, "pre", {}).pop(rid, None)


@pytest.fixture(scope="module")
def S():
    from paper_2504_18154_b200 import build
    build.build(verbose=False)
    from paper_2504_18154_b200 import serve
    return serve


def test_live_serving_completes_and_rolls(S):
    trace = make_trace("alpaca", 60, seed=3, rate_per_s=600.0, vocab=1000)
    for r in trace:
        r.output_len = min(r.output_len, 8)
    insts = [FakeInstance(scale=1.0) for _ in range(3)]
    srv = S.PaDGServer(insts, slo_ttft_ns=8_000_000, slo_tpot_ns=SEC // 50, reserve_tokens=32,
                       predictor_table=((16, 4096), (2_000_000, 60_000_000)), token_budget=4096)
    out = srv.run(trace, timeout_s=60)
    assert all(r.t_done_ns >= 0 for r in out.values()), "request lost"
    for r in out.values():
        assert r.n_gen == r.output_len if hasattr(r, "output_len") else r.n_gen == r.G
        assert len(r.tokens) == r.G
        assert r.arrival_ns <= r.t_first_ns <= r.t_decode_begin_ns <= r.t_done_ns
    used = {r.inst for r in out.values()}
    assert len(used) >= 2, "rolling activation should spread load over instances"
    # temporal disaggregation: every instance alternates prefill-only and decode-only phase calls
    for inst in insts:
        kinds = [c[0] for c in inst.calls]
        assert "prefill" in kinds and "decode" in kinds
    # routing log: every routed request went to exactly one instance
    routed = [x for x in srv.route_log if x[2] >= 0]
    assert sorted(x[1] for x in routed) == sorted(out)


def test_nodg_policy_round_robin_no_deferral(S):
    """NoDG separate batching (8(f) N3): immediate round-robin routing, every instance
    takes prefills interleaved with its decode steps, nothing is ever deferred."""
    trace = make_trace("alpaca", 40, seed=5, rate_per_s=400.0, vocab=1000)
    for r in trace:
        r.output_len = min(r.output_len, 6)
    insts = [FakeInstance(scale=1.0) for _ in range(3)]
    srv = S.PaDGServer(insts, slo_ttft_ns=8_000_000, slo_tpot_ns=SEC // 50, reserve_tokens=32,
                       predictor_table=((16, 4096), (2_000_000, 60_000_000)), token_budget=4096, policy="nodg")
    out = srv.run(trace, timeout_s=60)
    assert all(r.t_done_ns >= 0 for r in out.values())
    assert all(x[2] >= 0 for x in srv.route_log), "NoDG never defers"
    order = [x[2] for x in sorted(srv.route_log, key=lambda x: (x[0], x[1]))]
    by_arrival = sorted(out.values(), key=lambda r: (r.arrival_ns, r.req_id))
    assert [r.inst for r in by_arrival] == [i % 3 for i in range(len(by_arrival))]
    assert sorted(order) == sorted(r.inst for r in out.values())
    with pytest.raises(ValueError):
        S.PaDGServer(insts, 1, 1, 1, policy="tdpipe")


def test_sarathi_policy_hybrid_iterations(S):
    """NoDG hybrid batching (8(f) N3): every worker iteration is one hybrid step within
    the token budget; prompts longer than the budget are split into chunks."""
    trace = make_trace("alpaca", 30, seed=8, rate_per_s=300.0, vocab=1000)
    for r in trace:
        r.output_len = min(r.output_len, 5)
    insts = [FakeInstance(scale=1.0) for _ in range(2)]
    srv = S.PaDGServer(insts, slo_ttft_ns=8_000_000, slo_tpot_ns=SEC // 50, reserve_tokens=32,
                       predictor_table=((16, 4096), (2_000_000, 60_000_000)), token_budget=4096, policy="sarathi",
                       chunk_budget=48)
    out = srv.run(trace, timeout_s=60)
    assert all(r.t_done_ns >= 0 for r in out.values())
    for r in out.values():
        assert len(r.tokens) == r.G and r.t_first_ns == r.t_decode_begin_ns <= r.t_done_ns
    for inst in insts:
        assert inst.calls and all(c[0] == "hybrid" for c in inst.calls)
        assert all(c[3] <= 48 or c[1] == 0 for c in inst.calls)   # budget (decode-only calls may exceed)
    assert any(r.S > 48 for r in out.values())                    # some prompts needed several chunks


def test_product_metrics_match_oracle_definition():
    import random
    from oracle import metrics as OM
    from paper_2504_18154_b200 import metrics as MX
    rng = random.Random(4)
    for _ in range(2000):
        arr = rng.randint(0, 10 ** 9)
        tf = -1 if rng.random() < 0.05 else arr + rng.randint(0, 2 * 10 ** 9)
        db = tf + rng.randint(0, 10 ** 8) if tf >= 0 else -1
        G = rng.randint(1, 50)
        td = db + rng.randint(0, (G - 1) * 2 * 10 ** 8) if tf >= 0 else -1
        slo = (rng.choice([10 ** 9, 5 * 10 ** 8]), rng.choice([10 ** 8, 5 * 10 ** 7]))
        a = MX.request_ok(arr, tf, db, td, G, *slo)
        b = OM.request_metrics(arr, tf, db, td, G, *slo)
        assert a["ok"] == b.ok and a["finished"] == b.finished
        if b.finished:
            assert a["ttft_ok"] == b.ttft_ok and a["tpot_ok"] == b.tpot_ok
    assert MX.bisect_goodput(lambda r: 1.0 if r <= 13.0 else 0.0, 0.9, 1, 100, 20) == pytest.approx(13.0, abs=1e-3)


def test_worker_prefers_prefill_after_decode_step(S):
    """Intra-instance policy: a request arriving during decoding is
    prefilled right after the in-flight decode step (non-preemptive, A15)."""
    inst = FakeInstance(scale=1.0)
    srv = S.PaDGServer([inst], slo_ttft_ns=10 * SEC, slo_tpot_ns=SEC, reserve_tokens=16, token_budget=4096)
    trace = make_trace("tiny", 2, seed=1, vocab=1000)
    trace[0].arrival_ns, trace[0].output_len = 0, 30
    trace[1].arrival_ns, trace[1].output_len = 40_000_000, 3      # arrives ~40 ms later, mid-decode
    out = srv.run(trace, timeout_s=30)
    seq = [c[0] for c in inst.calls]
    i = seq.index("prefill", 1)
    assert seq[:i] == ["prefill"] + ["decode"] * (i - 1) and i > 1
    assert out[1].t_first_ns < out[0].t_done_ns


class FakeKVInstance(FakeInstance):
    """+ export_kv / import_kv (FuDG hand-off) with a per-request generation counter."""

    device = "cpu"

    def export_kv(self, rid, device):
        state = self.gen.pop(rid)
        self.calls.append(("export", 1))
        return (rid, state)

    def import_kv(self, handle):
        rid, state = handle
        assert rid not in self.gen
        self.gen[rid] = state
        self.calls.append(("import", 1))


def test_fudg_prefill_and_decode_roles(S):
    """FuDG baseline: prefill instances only prefill and hand every request's KV to a
    decode instance, which only decodes; every request completes with G tokens."""
    from paper_2504_18154_b200.serve import PaDGServer
    insts = [FakeKVInstance() for _ in range(3)]
    trace = make_trace("sharegpt", 40, seed=5, rate_per_s=200.0, vocab=1000)
    for r in trace:
        r.output_len = min(r.output_len, 24)
    srv = PaDGServer(insts, 5 * SEC, SEC // 10, reserve_tokens=64, policy="fudg", fudg_prefill=1)
    out = srv.run(trace, timeout_s=60)
    assert all(r.t_done_ns >= 0 and len(r.tokens) == r.G for r in out.values())
    assert {k for k, *_ in insts[0].calls} <= {"prefill", "export"}
    for d in insts[1:]:
        assert {k for k, *_ in d.calls} <= {"import", "decode"}
    n_multi = sum(1 for r in out.values() if r.G > 1)
    assert sum(1 for c in insts[0].calls if c[0] == "export") == n_multi
    assert sum(sum(1 for c in d.calls if c[0] == "import") for d in insts[1:]) == n_multi
    for r in out.values():
        assert r.t_first_ns <= r.t_decode_begin_ns <= r.t_done_ns


class FakeBlockInstance(FakeInstance):
    """+ the engine's 64-token KV block accounting: a prefill holds ceil(S/64) blocks, a
    decode step that writes position p needs ceil((p+1)/64); exceeding the pool raises
    like ECOSERVE_ERR_KV_EXHAUSTED. The prefill's prompt length is what the worker sends
    (prompt + generated tokens for a recompute)."""

    def __init__(self, num_blocks, **kw):
        super().__init__(num_blocks=num_blocks, **kw)
        self.kv = {}   # rid -> tokens with KV (prompt + fed tokens)
        self.prefills = []

    def used(self):
        return sum((n + 63) // 64 for n in self.kv.values())

    def prefill(self, reqs):
        for rid, p, g in reqs:
            assert g >= 1
            self.kv[rid] = len(p)
            self.prefills.append((rid, len(p), g))
        assert self.used() <= self.num_blocks, "KV pool exhausted at prefill"
        return super().prefill(reqs)

    def decode(self, ids, steps):
        toks, nf = super().decode(ids, steps)
        for i, rid in enumerate(ids):
            self.kv[rid] += int((toks[i] >= 0).sum())
        assert self.used() <= self.num_blocks, "KV pool exhausted at decode"
        return toks, nf

    def release(self, ids):
        super().release(ids)
        for rid in ids:
            self.kv.pop(rid, None)


def test_preempt_admission_recomputes_under_kv_pressure(S):
    """Reading A14 in live mode: with the reservation R = 0 the macro admits more than the
    pool holds once outputs grow; the worker preempts the latest arrivals before a decode
    step would outgrow the pool and re-prefills them with prompt + generated tokens. Every
    request still finishes with exactly G tokens and the pool never overflows."""
    trace = make_trace("tiny", 12, seed=6, rate_per_s=2000.0, vocab=1000)
    for r in trace:
        r.output_len = 60 + (r.req_id * 37) % 90
    inst = FakeBlockInstance(num_blocks=9, scale=1.0)
    srv = S.PaDGServer([inst], slo_ttft_ns=100 * SEC, slo_tpot_ns=100 * SEC, reserve_tokens=0, token_budget=4096,
                       admission="preempt")
    out = srv.run(trace, timeout_s=60)
    assert all(r.t_done_ns >= 0 and len(r.tokens) == r.G and r.n_gen == r.G for r in out.values())
    w = srv.workers[0]
    assert w.n_preempted >= 1
    recomputes = [(rid, n, g) for rid, n, g in inst.prefills if n > out[rid].S]
    assert len(recomputes) == w.n_preempted
    for rid, n, g in recomputes:          # prompt + every generated token, the rest still owed
        r = out[rid]
        assert n - r.S + g == r.G
    for r in out.values():
        assert r.arrival_ns <= r.t_first_ns <= r.t_decode_begin_ns <= r.t_done_ns
    with pytest.raises(ValueError):
        S.PaDGServer([inst], 1, 1, 0, policy="sarathi", admission="preempt")


def test_mitosis_resize_migrates_and_completes(S):
    """Mitosis live (8(f) N1): the macro starts with 2 of 4 instances, expands
    to 4, then contracts to 1 -- the contracted instances hand their prefilled requests
    over with the KV (export / import) and their queued ones as arrivals. Every request
    completes with its G tokens, in the same sequence as without migration; the router
    only uses the active prefix between resize events."""
    from paper_2504_18154_b200.serve import PaDGServer
    insts = [FakeKVInstance(scale=1.0) for _ in range(4)]
    trace = make_trace("alpaca", 90, seed=12, rate_per_s=200.0, vocab=1000)
    for r in trace:
        r.output_len = min(r.output_len, 24)
    srv = PaDGServer(insts, slo_ttft_ns=8_000_000, slo_tpot_ns=SEC // 50, reserve_tokens=32,
                     predictor_table=((16, 4096), (2_000_000, 60_000_000)), token_budget=4096,
                     resize=[(0, 2), (0.12, 4), (0.3, 1)])
    out = srv.run(trace, timeout_s=60)
    assert all(r.t_done_ns >= 0 and len(r.tokens) == r.G for r in out.values()), "request lost"
    for r in out.values():  # the fake's token k of request rid is (rid + k) % 997 wherever it ran
        assert r.tokens[0] == r.req_id % 997
        assert r.tokens[1:] == [(r.req_id + k) % 997 for k in range(1, r.G)]
    (t_grow, _, n1), (t_shrink, _, n2) = srv.resize_log[1], srv.resize_log[2]
    assert (n1, n2) == (4, 1)
    for t, rid, i in srv.route_log:
        if i >= 0 and t < t_grow:
            assert i < 2
        if i >= 0 and t >= t_shrink:
            assert i == 0
    assert sum(w.n_migrated_out for w in srv.workers[1:]) > 0, "contraction moved running requests"
    exports = sum(1 for d in insts[1:] for c in d.calls if c[0] == "export")
    imports = sum(1 for c in insts[0].calls if c[0] == "import")
    assert exports == imports == sum(w.n_migrated_out for w in srv.workers)
    for r in out.values():  # timestamps stay ordered across a move (TPOT counts from the decode start)
        assert r.arrival_ns <= r.t_first_ns <= r.t_decode_begin_ns <= r.t_done_ns
    for d in insts:
        assert not d.gen, "every request released"


def test_mitosis_auto_triggers(S):
    """Mitosis triggers: a burst that no single instance can admit under the TTFT
    SLO keeps requests Deferred -> the macro expands; a later quiet period -> it contracts.
    Every request completes with its token sequence."""
    from paper_2504_18154_b200.serve import PaDGServer
    insts = [FakeKVInstance(scale=1.0) for _ in range(4)]
    burst = make_trace("alpaca", 120, seed=31, rate_per_s=1500.0, vocab=1000)
    late = make_trace("alpaca", 6, seed=32, rate_per_s=20.0, vocab=1000)
    for k, r in enumerate(late):
        r.req_id = 1000 + k
        r.arrival_ns += int(0.5 * SEC)
    trace = burst + late
    for r in trace:
        r.output_len = min(r.output_len, 24)
    srv = PaDGServer(insts, slo_ttft_ns=8_000_000, slo_tpot_ns=SEC // 50, reserve_tokens=32,
                     predictor_table=((16, 4096), (2_000_000, 60_000_000)), token_budget=4096,
                     resize=dict(n_min=1, n_max=4, n_start=1, up_s=0.01, down_s=0.15, down_live=4,
                                 cooldown_s=0.02))
    out = srv.run(trace, timeout_s=60)
    assert all(r.t_done_ns >= 0 and len(r.tokens) == r.G for r in out.values())
    for r in out.values():
        assert r.tokens[1:] == [(r.req_id + k) % 997 for k in range(1, r.G)]
    sizes = [b for _, _, b in srv.resize_log]
    assert max(sizes) > 1, f"the burst expanded the macro: {srv.resize_log}"
    peak = sizes.index(max(sizes))
    assert min(sizes[peak:]) < max(sizes), f"the quiet period contracted it: {srv.resize_log}"
    for d in insts:
        assert not d.gen
