"""ORACLE (test infrastructure only) -- the macro-instance scheduler, SURVEY 8(c) C5.

* Alg. 1 InterSchedule (prose P:556-559): try the instance
  the previous request went to; if CheckConstraints fails, probe the next ones
  cyclically (prose reading A9; the printed variant is kept as ``probe="printed"``),
  at most one full cycle; Deferred if none passes.
* Alg. 2 CheckConstraints (prose P:561-567), all times int64 ns:
    C1 TTFT : Pending = {r : r.arrival >= t_switch or r.t_first unset} + {req}
              (A11); t_total = sum pred(r.S); fail iff t_total > SLO_TTFT.
    C2 TPOT : Existed = {r : r.arrival < t_switch, t_first set, unfinished};
              saved_r = r.n_generated * SLO_TPOT - (now - r.t_first)  (A10);
              fail iff sum(saved) < |Existed| * t_total  (== mean < t_total).
    C3 KV   : committed = sum_r max(ceil((S+R)/64), ceil((S+n_gen)/64)) (A14);
              fail iff ceil((req.S+R)/64) > total_blocks - committed.
  Boundary comparisons per A12 (equality passes).
* Prefill predictor ("predicted in advance by profiling"): either the
  fixed integer cost model of SURVEY 8(c) (DES / parity) or a piecewise-linear
  table over profiled (S, ns) samples (live mode, A13).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

BLOCK_TOKENS = 64

OK, FAIL_TTFT, FAIL_TPOT, FAIL_KV = 0, 1, 2, 3
DEFERRED = -1


def ceil_div(a: int, b: int) -> int:
    return -(-a // b)


@dataclass(frozen=True)
class CostModel:
    """Fixed integer cost model. b, c, f in picoseconds."""
    a: int = 2_000_000        # ns per prefill request
    b: int = 14_320_000       # ps per prompt token
    c: int = 270              # ps per prompt token^2
    d: int = 3_280_000        # ns per decode step
    e: int = 1_000            # ns per decode row
    f: int = 28_600           # ps per context token in the step

    def prefill_ns(self, S: int) -> int:
        return self.a + (self.b * S + self.c * S * S) // 1000

    def decode_ns(self, B: int, sum_ctx: int) -> int:
        return self.d + self.e * B + (self.f * sum_ctx) // 1000


@dataclass(frozen=True)
class TablePredictor:
    """Piecewise-linear prefill predictor over sorted (S, ns) samples (A13).
    Outside the sampled range the nearest segment is extended."""
    lens: Tuple[int, ...]
    ns: Tuple[int, ...]

    def prefill_ns(self, S: int) -> int:
        L, N = self.lens, self.ns
        if len(L) == 1:
            return N[0]
        i = 0
        while i < len(L) - 2 and S > L[i + 1]:
            i += 1
        dx = L[i + 1] - L[i]
        num = (N[i + 1] - N[i]) * (S - L[i])
        # floor division toward -inf, identical in the C++ implementation
        return N[i] + num // dx


@dataclass
class ReqStatus:
    req_id: int
    arrival_ns: int
    prompt_len: int
    t_first_ns: int = -1       # -1: first token not produced yet
    n_generated: int = 0
    finished: bool = False


@dataclass
class InstStatus:
    phase: int = 0             # 0 idle, 1 prefill, 2 decode
    t_switch_ns: int = 0       # A18: initial t_switch = 0
    total_blocks: int = 0
    alive: bool = True
    reqs: Dict[int, ReqStatus] = field(default_factory=dict)


@dataclass(frozen=True)
class MacroConfig:
    slo_ttft_ns: int
    slo_tpot_ns: int
    reserve_tokens: int        # R of reading A14
    probe: str = "cycle"       # "cycle" (prose, A9) | "printed" (Alg. 1 as printed)


def check_constraints(st: InstStatus, req_S: int, req_arrival: int, now: int,
                      cfg: MacroConfig, pred) -> int:
    """Alg. 2. Returns OK or the first failing constraint."""
    if not st.alive:
        return FAIL_KV  # a dead instance offers no capacity (failure detection)
    # Constraint 1: TTFT
    pending = [r for r in st.reqs.values()
               if not r.finished and (r.arrival_ns >= st.t_switch_ns or r.t_first_ns < 0)]
    t_total = sum(pred.prefill_ns(r.prompt_len) for r in pending) + pred.prefill_ns(req_S)
    if t_total > cfg.slo_ttft_ns:
        return FAIL_TTFT
    # Constraint 2: TPOT (typewriter mode)
    existed = [r for r in st.reqs.values()
               if not r.finished and r.arrival_ns < st.t_switch_ns and r.t_first_ns >= 0]
    if existed:
        saved = [r.n_generated * cfg.slo_tpot_ns - (now - r.t_first_ns) for r in existed]
        if sum(saved) < len(existed) * t_total:
            return FAIL_TPOT
    # Constraint 3: KV cache capacity
    R = cfg.reserve_tokens
    committed = sum(max(ceil_div(r.prompt_len + R, BLOCK_TOKENS),
                        ceil_div(r.prompt_len + r.n_generated, BLOCK_TOKENS))
                    for r in st.reqs.values() if not r.finished)
    if ceil_div(req_S + R, BLOCK_TOKENS) > st.total_blocks - committed:
        return FAIL_KV
    return OK


class Macro:
    """A macro instance: the smallest scheduling unit."""

    def __init__(self, n_inst: int, total_blocks: Sequence[int], cfg: MacroConfig, pred):
        self.cfg = cfg
        self.pred = pred
        self.status = [InstStatus(total_blocks=int(b)) for b in total_blocks]
        self.prev_idx = 0          # A18
        self.deferred: List[Tuple[int, int, int]] = []   # FIFO of (req_id, S, arrival)
        self.log: List[Tuple] = []  # (now, req_id, chosen, [outcome per probed instance])

    @property
    def n(self) -> int:
        return len(self.status)

    def route(self, req_id: int, S: int, arrival: int, now: int) -> int:
        """Alg. 1. On success the request is recorded as pending in the
        macro's view of the chosen instance and prev_idx moves to it."""
        outcomes = []
        if self.cfg.probe == "printed":
            i = self.prev_idx
            res = check_constraints(self.status[i], S, arrival, now, self.cfg, self.pred)
            outcomes.append(res)
            chosen = i if res == OK else (i + 1) % self.n
        else:
            chosen = DEFERRED
            for k in range(self.n):
                i = (self.prev_idx + k) % self.n
                res = check_constraints(self.status[i], S, arrival, now, self.cfg, self.pred)
                outcomes.append(res)
                if res == OK:
                    chosen = i
                    break
        self.log.append((now, req_id, chosen, tuple(outcomes)))
        if chosen == DEFERRED:
            return DEFERRED
        self.prev_idx = chosen
        self.status[chosen].reqs[req_id] = ReqStatus(req_id, arrival, S)
        return chosen

    def update_status(self, i: int, phase: int, t_switch: int, reqs: Sequence[ReqStatus],
                      total_blocks: Optional[int] = None, alive: bool = True) -> None:
        """Status push from instance i: entries overwrite the
        macro's view by req_id; finished requests are dropped."""
        st = self.status[i]
        st.phase, st.t_switch_ns, st.alive = phase, t_switch, alive
        if total_blocks is not None:
            st.total_blocks = total_blocks
        for r in reqs:
            if r.finished:
                st.reqs.pop(r.req_id, None)
            else:
                st.reqs[r.req_id] = ReqStatus(r.req_id, r.arrival_ns, r.prompt_len,
                                              r.t_first_ns, r.n_generated, False)

    def drain_deferred(self, now: int) -> List[Tuple[int, int]]:
        """Retry the deferred FIFO in order, stopping at the first request that
        is still Deferred (head-of-line order is preserved)."""
        out = []
        while self.deferred:
            rid, S, arr = self.deferred[0]
            i = self.route(rid, S, arr, now)
            if i == DEFERRED:
                break
            self.deferred.pop(0)
            out.append((rid, i))
        return out
