"""ORACLE (test infrastructure only) -- per-request metrics and goodput, SURVEY 8(c) C6.

* Sec. 3.3: the reported TTFT includes the phase-switching wait of
  the prefill phase (TTFT = t_first - arrival); TPOT is measured after the
  switch delay: TPOT = (t_done - t_decode_begin) / (G - 1) (reading A7: G counts
  the prefill token). A G = 1 request is TPOT-ok.
* Typewriter mode: TPOT-ok iff t_done - t_decode_begin <= (G-1) SLO_TPOT.
* Attainment: fraction of requests meeting TTFT and TPOT jointly; unfinished
  requests count as violations. A run passes percentile p iff
  attainment >= p.
* Goodput: the largest Poisson rate whose run passes p, found by bisection
  ("incrementally increasing the request rate until the system fails").
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Iterable


@dataclass
class ReqMetrics:
    ttft_ns: int
    switch_wait_ns: int
    tpot_ns: float
    ttft_ok: bool
    tpot_ok: bool
    finished: bool

    @property
    def ok(self) -> bool:
        return self.finished and self.ttft_ok and self.tpot_ok


def request_metrics(arrival_ns: int, t_first_ns: int, t_decode_begin_ns: int, t_done_ns: int,
                    G: int, slo_ttft_ns: int, slo_tpot_ns: int) -> ReqMetrics:
    if t_first_ns < 0 or t_done_ns < 0:
        return ReqMetrics(-1, -1, float("nan"), False, False, False)
    ttft = t_first_ns - arrival_ns
    if G <= 1:
        return ReqMetrics(ttft, 0, 0.0, ttft <= slo_ttft_ns, True, True)
    span = t_done_ns - t_decode_begin_ns
    return ReqMetrics(ttft, t_decode_begin_ns - t_first_ns, span / (G - 1),
                      ttft <= slo_ttft_ns, span <= (G - 1) * slo_tpot_ns, True)


def attainment(ms: Iterable[ReqMetrics]) -> float:
    ms = list(ms)
    if not ms:
        raise ValueError("attainment of an empty run")
    return sum(1 for m in ms if m.ok) / len(ms)


def passes(ms, p: float) -> bool:
    return attainment(ms) >= p


def goodput(run_at_rate: Callable[[float], float], p: float, lo: float, hi: float, iters: int = 12) -> float:
    """Bisection for the largest rate in [lo, hi] whose attainment >= p.
    `run_at_rate(rate)` returns the attainment of an independent run."""
    if lo >= hi:
        raise ValueError("rate bounds inverted")
    if run_at_rate(lo) < p:
        return 0.0
    if run_at_rate(hi) >= p:
        return hi
    for _ in range(iters):
        mid = 0.5 * (lo + hi)
        if run_at_rate(mid) >= p:
            lo = mid
        else:
            hi = mid
    return lo
