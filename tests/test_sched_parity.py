"""Bit-exact parity of the C++ macro scheduler (libecoserve.so) with the oracle
("routing/phase decisions must be bit-exact"). CPU only."""
import random

import numpy as np
import pytest

from oracle import des, scheduler as S
from synthetic.traces import Request, make_trace

SEC = 1_000_000_000


@pytest.fixture(scope="module")
def M():
    from paper_2504_18154_b200 import build, macro
    build.build(verbose=False)
    return macro


def test_check_constraints_bitexact_random(M):
    rng = random.Random(5)
    outcomes = set()
    for trial in range(400):
        n_inst = rng.randint(1, 4)
        blocks = [rng.randint(0, 400) for _ in range(n_inst)]
        slo_ttft = rng.choice([SEC // 10, SEC // 4, SEC, 5 * SEC])
        R = rng.choice([0, 64, 256])
        table = None
        if rng.random() < 0.3:
            lens = sorted(rng.sample(range(1, 5000), 4))
            table = (lens, sorted(rng.randint(1_000_000, 90_000_000) for _ in range(4)))
        cfg = M.SchedConfig(n_inst, slo_ttft, SEC // 10, R, blocks, table=table)
        cm = M.MacroScheduler(cfg)
        pred = S.TablePredictor(tuple(table[0]), tuple(table[1])) if table else S.CostModel()
        om = S.Macro(n_inst, blocks, S.MacroConfig(slo_ttft, SEC // 10, R), pred)
        for i in range(n_inst):
            t_switch = rng.randint(0, 10 * SEC)
            reqs = []
            for k in range(rng.randint(0, 8)):
                arr = rng.randint(0, 15 * SEC)
                tf = -1 if rng.random() < 0.3 else arr + rng.randint(0, SEC)
                reqs.append((100 * i + k, arr, rng.randint(1, 4096), tf, 0 if tf < 0 else rng.randint(1, 300),
                             rng.random() < 0.1))
            cm.update_status(i, 2, t_switch, blocks[i], reqs)
            om.update_status(i, 2, t_switch, [S.ReqStatus(*r) for r in reqs])
        for q in range(5):
            now = rng.randint(10 * SEC, 16 * SEC)
            S_ = rng.randint(1, 4096)
            for i in range(n_inst):
                a = cm.check(i, S_, now, now)
                b = S.check_constraints(om.status[i], S_, now, now, om.cfg, pred)
                assert a == b
                outcomes.add(a)
            got = cm.route(1000 + q, now, S_, now)
            ref = om.route(1000 + q, S_, now, now)
            assert got[0] == ref and tuple(got[1]) == om.log[-1][3]
            assert cm.prev_idx == om.prev_idx
            if table:
                assert cm.predict_prefill_ns(S_) == pred.prefill_ns(S_)
    assert outcomes == {0, 1, 2, 3}


@pytest.mark.parametrize("preset,rate,n_inst,seed", [("sharegpt", 60.0, 4, 1), ("sharegpt", 200.0, 4, 2),
                                                     ("alpaca", 300.0, 2, 3), ("8b-cycle", 8.0, 3, 4),
                                                     ("long", 3.0, 4, 5)])
@pytest.mark.parametrize("probe", ["cycle", "printed"])
def test_des_bitexact_vs_oracle(M, preset, rate, n_inst, seed, probe):
    reqs = make_trace(preset, 250, seed=seed, rate_per_s=rate)
    R = max(r.output_len for r in reqs)
    blocks = 9000
    ocfg = S.MacroConfig(5 * SEC, SEC // 10, R, probe=probe)
    sim = des.simulate(reqs, n_inst, blocks, ocfg, S.CostModel(), 16384)
    cfg = M.SchedConfig(n_inst, 5 * SEC, SEC // 10, R, [blocks] * n_inst, probe_printed=(probe == "printed"))
    got = M.des_run(cfg, [r.arrival_ns for r in reqs], [r.prompt_len for r in reqs], [r.output_len for r in reqs])
    for k, r in enumerate(reqs):
        o = sim.reqs[r.req_id]
        assert (got["inst"][k], got["t_first"][k], got["t_decode_begin"][k], got["t_done"][k]) == \
            (o.inst, o.t_first_ns, o.t_decode_begin_ns, o.t_done_ns), k
    assert got["route_log"] == [tuple(x) for x in sim.route_log]


def test_deferred_fifo_drain(M):
    cfg = M.SchedConfig(2, 100_000_000, SEC // 10, 0, [1000, 1000], cost_a_ns=60_000_000, cost_b_ps=0, cost_c_ps=0)
    cm = M.MacroScheduler(cfg)
    assert cm.route(1, 0, 10, 0)[0] == 0
    assert cm.route(2, 0, 10, 0)[0] == 1
    inst, outc = cm.route(3, 0, 10, 0)
    assert inst == -1 and outc == [1, 1]       # both fail TTFT (2 x 60 ms > 100 ms)
    cm.defer(3, 0, 10)
    cm.defer(4, 0, 10)
    assert cm.drain_deferred(1) == []
    cm.update_status(1, 1, 0, 1000, [(2, 0, 10, 5, 1, True)])   # request 2 finished
    assert cm.drain_deferred(2) == [(3, 1)]    # 3 fits, 4 is still deferred (FIFO head stops)


@pytest.mark.parametrize("seed", range(8))
def test_des_preemption_bitexact_vs_oracle(M, seed):
    """Reading A14 under KV pressure (R = 0 on a small pool): the C++ DES preempts and
    recomputes exactly as the oracle does (timestamps, routing, preemption counts)."""
    rng = random.Random(7000 + seed)
    n = rng.randint(6, 40)
    arr = sorted(rng.randint(0, 2 * SEC) for _ in range(n))
    reqs = [Request(i, arr[i], rng.randint(16, 600), rng.randint(20, 400)) for i in range(n)]
    n_inst, blocks = rng.randint(1, 3), rng.choice([18, 24, 40])
    ocfg = S.MacroConfig(50 * SEC, SEC, 0)
    sim = des.simulate(reqs, n_inst, blocks, ocfg, S.CostModel(), 2048)
    assert sim.preempt_log, "the case must exercise A14"
    cfg = M.SchedConfig(n_inst, 50 * SEC, SEC, 0, [blocks] * n_inst)
    got = M.des_run(cfg, [r.arrival_ns for r in reqs], [r.prompt_len for r in reqs], [r.output_len for r in reqs],
                    token_budget=2048)
    for k, r in enumerate(reqs):
        o = sim.reqs[r.req_id]
        assert (got["inst"][k], got["t_first"][k], got["t_decode_begin"][k], got["t_done"][k],
                got["n_preempt"][k]) == (o.inst, o.t_first_ns, o.t_decode_begin_ns, o.t_done_ns, o.n_preempt), k
    assert got["route_log"] == [tuple(x) for x in sim.route_log]
