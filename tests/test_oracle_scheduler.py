"""Pins of the scheduler / DES / metrics oracle."""
import json
import os
import random
from fractions import Fraction

import pytest

from oracle import des, metrics, scheduler as S, tick_sim
from synthetic.traces import Request, make_trace

GOLD = os.path.join(os.path.dirname(__file__), "golden")
spec = json.load(open(os.path.join(GOLD, "spec_examples.json")))
SEC = 1_000_000_000


class PerToken:
    """Predictor used by the worked examples: 1 ms per prompt token."""
    def prefill_ns(self, s):
        return s * 1_000_000


CFG = S.MacroConfig(slo_ttft_ns=5 * SEC, slo_tpot_ns=SEC // 10, reserve_tokens=64)


def test_spec_check_constraints_examples():
    ex = spec["check_constraints"]
    st = S.InstStatus(total_blocks=1000)
    cfg = S.MacroConfig(int(ex["idle"]["slo_ttft_s"] * SEC), SEC // 10, 64)
    assert S.check_constraints(st, 200, 0, 0, cfg, PerToken()) == S.OK
    # pending predicted 4.9 s, new request 0.2 s, SLO 5 s -> TTFT fails (5.1 > 5)
    st = S.InstStatus(total_blocks=1000, t_switch_ns=0)
    st.reqs[1] = S.ReqStatus(1, 10, 4900)
    assert S.check_constraints(st, 200, 20, 20, CFG, PerToken()) == S.FAIL_TTFT
    # saved = 100 * 0.1 - 8 = 2 s >= t_total = 1.5 s -> TPOT passes
    now = 100 * SEC
    st = S.InstStatus(total_blocks=1000, t_switch_ns=now - SEC)
    st.reqs[1] = S.ReqStatus(1, 0, 10, t_first_ns=now - 8 * SEC, n_generated=100)
    assert S.check_constraints(st, 1500, now, now, CFG, PerToken()) == S.OK
    # ... and fails when t_total exceeds the 2 s of saved TPOT
    assert S.check_constraints(st, 2001, now, now, CFG, PerToken()) == S.FAIL_TPOT
    # boundary (A12): saved == t_total passes
    assert S.check_constraints(st, 2000, now, now, CFG, PerToken()) == S.OK


def test_kv_constraint_boundary():
    st = S.InstStatus(total_blocks=10)
    st.reqs[1] = S.ReqStatus(1, 0, 100)                 # commits ceil((100+64)/64) = 3 blocks
    cfg = S.MacroConfig(100 * SEC, SEC, 64)
    assert S.check_constraints(st, 384, 0, 0, cfg, PerToken()) == S.OK      # ceil(448/64) = 7 == 10-3
    assert S.check_constraints(st, 385, 0, 0, cfg, PerToken()) == S.FAIL_KV


def test_spec_inter_schedule_examples():
    m = S.Macro(3, [1000] * 3, CFG, PerToken())
    assert m.route(1, 100, 0, 0) == 0 and m.prev_idx == 0          # fresh -> 0
    # saturate instance 0's TTFT budget
    m.status[0].reqs[1].prompt_len = 4950
    assert m.route(2, 100, 1, 1) == 1 and m.prev_idx == 1          # -> 1
    for i in range(3):
        m.status[i].reqs[100 + i] = S.ReqStatus(100 + i, 1, 5000)
    assert m.route(3, 100, 2, 2) == S.DEFERRED                      # all fail
    assert m.prev_idx == 1


def brute_check(st, req_S, now, cfg, pred):
    """Independent re-evaluation of Alg. 2 with exact rationals and a mean."""
    live = [r for r in st.reqs.values() if not r.finished]
    pending = [r for r in live if r.arrival_ns >= st.t_switch_ns or r.t_first_ns == -1]
    t_total = Fraction(sum(pred.prefill_ns(r.prompt_len) for r in pending) + pred.prefill_ns(req_S))
    if t_total > cfg.slo_ttft_ns:
        return S.FAIL_TTFT
    existed = [r for r in live if r not in pending]
    if existed:
        mean = Fraction(sum(r.n_generated * cfg.slo_tpot_ns - (now - r.t_first_ns) for r in existed), len(existed))
        if mean < t_total:
            return S.FAIL_TPOT
    import math
    need = lambda n: math.ceil(Fraction(n, 64))  # noqa: E731
    committed = sum(max(need(r.prompt_len + cfg.reserve_tokens), need(r.prompt_len + r.n_generated)) for r in live)
    return S.FAIL_KV if need(req_S + cfg.reserve_tokens) > st.total_blocks - committed else S.OK


def test_check_constraints_vs_bruteforce_random():
    rng = random.Random(11)
    pred = S.CostModel()
    outcomes = set()
    for _ in range(1500):
        st = S.InstStatus(total_blocks=rng.randint(0, 400), t_switch_ns=rng.randint(0, 10 * SEC))
        now = st.t_switch_ns + rng.randint(0, 5 * SEC)
        for k in range(rng.randint(0, 8)):
            arr = rng.randint(0, now)
            tf = -1 if rng.random() < 0.3 else rng.randint(arr, now)
            st.reqs[k] = S.ReqStatus(k, arr, rng.randint(1, 4096), tf,
                                     0 if tf < 0 else rng.randint(1, 300), rng.random() < 0.1)
        cfg = S.MacroConfig(rng.choice([SEC // 10, SEC // 4, SEC, 5 * SEC]), SEC // 10, rng.choice([0, 64, 256]))
        req_S = rng.randint(1, 4096)
        got = S.check_constraints(st, req_S, now, now, cfg, pred)
        assert got == brute_check(st, req_S, now, cfg, pred)
        outcomes.add(got)
    assert outcomes == {S.OK, S.FAIL_TTFT, S.FAIL_TPOT, S.FAIL_KV}   # every branch exercised


def test_cost_model_defaults_match_roofline_derivation():
    c = S.CostModel()
    # 8B prefill at 60% of 1624.4 TF/s: 2*6.98e9 FLOP / 974.6e12 = 14.3 us per token
    assert abs(c.b / 1e3 - 2 * 6.98e9 / (0.6 * 1624.4e12) * 1e9) < 0.05 * c.b / 1e3
    # decode: 15.0 GB of weights at 70% of 6543.7 GB/s -> 3.28 ms
    assert abs(c.d - 15.0e9 / (0.7 * 6543.7e9) * 1e9) < 0.01 * c.d
    assert c.prefill_ns(1000) == 2_000_000 + (14_320_000 * 1000 + 270 * 10 ** 6) // 1000


def test_table_predictor_interpolation():
    p = S.TablePredictor((128, 512, 2048), (1000, 3000, 9000))
    assert p.prefill_ns(128) == 1000 and p.prefill_ns(512) == 3000 and p.prefill_ns(2048) == 9000
    assert p.prefill_ns(320) == 2000
    assert p.prefill_ns(4096) == 9000 + (6000 * 2048) // 1536    # last segment extended
    assert p.prefill_ns(0) == 1000 + (2000 * -128) // 384 == 333   # floor toward -inf


def single(reqs, n_inst=1, blocks=10_000, cfg=CFG, cost=None, budget=16384):
    return des.simulate(reqs, n_inst, blocks, cfg, cost or S.CostModel(), budget)


def test_des_single_request_closed_form():
    c = S.CostModel()
    r = Request(0, 1000, 300, 4)
    sim = single([r])
    rec = sim.reqs[0]
    assert rec.t_first_ns == 1000 + c.prefill_ns(300)
    assert rec.t_decode_begin_ns == rec.t_first_ns
    t = rec.t_first_ns
    for k in range(1, 4):
        t += c.decode_ns(1, 300 + k)
    assert rec.t_done_ns == t and rec.n_gen == 4


def test_des_request_arriving_mid_decode_waits_for_window():
    c = S.CostModel()
    r0 = Request(0, 0, 100, 50)
    sim0 = single([r0])
    t_mid = sim0.reqs[0].t_first_ns + c.decode_ns(1, 101) // 2      # inside the first decode step
    sim = single([r0, Request(1, t_mid, 200, 2)])
    rec = sim.reqs[1]
    step_end = sim.reqs[0].t_first_ns + c.decode_ns(1, 101)
    assert rec.t_first_ns == step_end + c.prefill_ns(200)             # A15 non-preemptive
    assert metrics.request_metrics(rec.arrival_ns, rec.t_first_ns, rec.t_decode_begin_ns, rec.t_done_ns,
                                   2, CFG.slo_ttft_ns, CFG.slo_tpot_ns).ttft_ns >= c.prefill_ns(200)


@pytest.mark.parametrize("seed", range(12))
def test_des_equals_tick_simulator(seed):
    rng = random.Random(seed)
    tick = 500_000
    cost = S.CostModel(a=rng.choice([1, 2]) * tick, b=tick * 1000 // 64 * rng.choice([1, 2]), c=0,
                       d=rng.choice([3, 5]) * tick, e=0, f=0)
    n_inst = rng.randint(1, 3)
    reqs = []
    for i in range(rng.randint(1, 8)):
        reqs.append(Request(i, rng.randint(0, 40) * tick, rng.choice([64, 128, 256, 512]), rng.randint(1, 12)))
    cfg = S.MacroConfig(slo_ttft_ns=rng.choice([20, 40, 80]) * tick, slo_tpot_ns=rng.choice([2, 6]) * tick,
                        reserve_tokens=16)
    blocks = rng.choice([12, 40])
    budget = rng.choice([256, 1024])
    sim = des.simulate(reqs, n_inst, blocks, cfg, cost, budget)
    recs, log, pre = tick_sim.tick_simulate(reqs, n_inst, blocks, cfg, cost, budget, tick, horizon=10 ** 13)
    assert pre == sim.preempt_log
    for rid, r in sim.reqs.items():
        t = recs[rid]
        assert (r.inst, r.t_first_ns, r.t_decode_begin_ns, r.t_done_ns, r.n_gen) == \
            (t["inst"], t["t_first_ns"], t["t_decode_begin_ns"], t["t_done_ns"], t["n_gen"])
    assert sim.route_log == log


def _pressure_case(seed):
    """A tiny trace whose outputs outgrow the reservation (R = 0): C3 admits more
    than the pool can hold once the requests grow, so A14 preemption must fire."""
    rng = random.Random(1000 + seed)
    tick = 500_000
    # one tick per prompt token, so recompute prefills (prompt + generated) stay on the tick grid
    cost = S.CostModel(a=rng.choice([1, 2]) * tick, b=tick * 1000, c=0, d=rng.choice([3, 5]) * tick, e=0, f=0)
    n_inst = rng.randint(1, 2)
    reqs = [Request(i, rng.randint(0, 30) * tick, rng.randint(20, 150), rng.randint(30, 160))
            for i in range(rng.randint(3, 8))]
    cfg = S.MacroConfig(slo_ttft_ns=10 ** 12, slo_tpot_ns=10 ** 12, reserve_tokens=0)
    blocks = rng.choice([6, 8, 10])
    return reqs, n_inst, blocks, cfg, cost, tick


@pytest.mark.parametrize("seed", range(16))
def test_des_preemption_equals_tick_simulator(seed):
    """Reading A14 (recompute preemption, TD-Pipe P:1112) in the DES == the naive
    tick simulator, bit-exact: timestamps, routing and the preemption log."""
    reqs, n_inst, blocks, cfg, cost, tick = _pressure_case(seed)
    sim = des.simulate(reqs, n_inst, blocks, cfg, cost, 256)
    recs, log, pre = tick_sim.tick_simulate(reqs, n_inst, blocks, cfg, cost, 256, tick, horizon=10 ** 13)
    assert pre == sim.preempt_log
    assert sim.route_log == log
    for rid, r in sim.reqs.items():
        t = recs[rid]
        assert (r.inst, r.t_first_ns, r.t_decode_begin_ns, r.t_done_ns, r.n_gen) == \
            (t["inst"], t["t_first_ns"], t["t_decode_begin_ns"], t["t_done_ns"], t["n_gen"])
        assert r.n_gen == r.G and r.t_done_ns >= 0                     # nothing lost, exact lengths
        assert r.arrival_ns <= r.t_first_ns <= r.t_decode_begin_ns <= r.t_done_ns
    assert max(sim.max_blocks_used) <= blocks                          # KV conservation


def test_preemption_fires_and_recomputes():
    """The pressure cases really exercise A14: requests are preempted, re-prefilled
    with prompt + generated tokens, and still finish with exactly G tokens."""
    fired = 0
    for seed in range(16):
        reqs, n_inst, blocks, cfg, cost, _ = _pressure_case(seed)
        sim = des.simulate(reqs, n_inst, blocks, cfg, cost, 256)
        fired += len(sim.preempt_log)
        for (t, rid, i) in sim.preempt_log:
            r = sim.reqs[rid]
            assert r.n_preempt >= 1 and r.t_first_ns <= t < r.t_done_ns and r.inst == i
    assert fired >= 10


def test_no_preemption_when_reservation_covers_outputs():
    """With R >= every output length, C3 keeps the pool from ever running out: the
    A14 path never fires (the parity runs rely on this)."""
    reqs = make_trace("sharegpt", 300, seed=2, rate_per_s=150.0)
    R = max(r.output_len for r in reqs)
    sim = des.simulate(reqs, 2, 3000, S.MacroConfig(5 * SEC, SEC // 10, reserve_tokens=R), S.CostModel(), 16384)
    assert sim.preempt_log == [] and all(r.t_done_ns >= 0 for r in sim.reqs.values())


def test_des_invariants_on_sharegpt_trace():
    reqs = make_trace("sharegpt", 300, seed=1, rate_per_s=100.0)
    cfg = S.MacroConfig(5 * SEC, SEC // 10, reserve_tokens=4096)
    sim = des.simulate(reqs, 4, 6000, cfg, S.CostModel(), 16384)
    done = 0
    for rid, r in sim.reqs.items():
        assert r.t_done_ns >= 0, "request lost"
        assert r.arrival_ns <= r.t_first_ns <= r.t_decode_begin_ns <= r.t_done_ns
        done += 1
    assert done == 300
    # routing locality: prev_idx changes only after a constraint failure
    prev = 0
    assert sim.macro.log
    for (t, rid, chosen, outcomes) in sim.macro.log:
        if chosen not in (S.DEFERRED, prev):
            assert outcomes[0] != S.OK
        if chosen != S.DEFERRED:
            # the chosen instance is the first feasible one in cyclic order
            assert all(o != S.OK for o in outcomes[:-1]) and outcomes[-1] == S.OK
            prev = chosen
    # rolling activation: prefill windows are staggered, every instance served requests
    assert len({r.inst for r in sim.reqs.values()}) == 4


def test_metrics_attainment_examples():
    ex = spec["attainment"]
    ms = [metrics.ReqMetrics(1, 0, 0.0, True, True, True)] * ex["ok"] + \
         [metrics.ReqMetrics(1, 0, 0.0, False, True, True)] * (ex["n"] - ex["ok"])
    assert metrics.passes(ms, 0.9) and not metrics.passes(ms, 0.99)
    m = metrics.request_metrics(0, 10, 25, 25 + 3 * 100, 4, 100, 100)
    assert m.ok and m.switch_wait_ns == 15 and m.tpot_ns == 100.0
    assert not metrics.request_metrics(0, 10, 25, 25 + 3 * 100 + 1, 4, 100, 100).tpot_ok
    assert not metrics.request_metrics(0, -1, -1, -1, 4, 100, 100).ok   # unfinished = violation
    assert metrics.request_metrics(0, 10, 10, 10, 1, 100, 1).tpot_ok    # G = 1


def test_goodput_bisection_monotone():
    gp = metrics.goodput(lambda rate: 1.0 if rate <= 7.25 else 0.5, 0.9, 1.0, 20.0, iters=20)
    assert abs(gp - 7.25) < 1e-4
