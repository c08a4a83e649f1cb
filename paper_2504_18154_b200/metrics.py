"""Serving metrics of the live PaDG server.

Sec. 3.3: the reported TTFT = t_first - arrival includes
the phase-switching wait; TPOT is measured after the switch delay:
TPOT = (t_done - t_decode_begin) / (G - 1), G counting the prefill token (A7);
typewriter mode: TPOT-ok iff t_done - t_decode_begin <= (G-1) SLO_TPOT.
Attainment counts requests meeting TTFT and TPOT jointly; unfinished requests
are violations. Goodput: the largest request rate whose attainment
reaches the percentile p.
"""
from __future__ import annotations

from typing import Callable, Dict, Iterable


def request_ok(arrival_ns: int, t_first_ns: int, t_decode_begin_ns: int, t_done_ns: int, G: int,
               slo_ttft_ns: int, slo_tpot_ns: int) -> Dict:
    if t_first_ns < 0 or t_done_ns < 0:
        return {"finished": False, "ttft_ok": False, "tpot_ok": False, "ok": False}
    ttft = t_first_ns - arrival_ns
    ttft_ok = ttft <= slo_ttft_ns
    if G <= 1:
        tpot_ok, tpot = True, 0.0
    else:
        span = t_done_ns - t_decode_begin_ns
        tpot_ok, tpot = span <= (G - 1) * slo_tpot_ns, span / (G - 1)
    return {"finished": True, "ttft_ns": ttft, "switch_wait_ns": t_decode_begin_ns - t_first_ns, "tpot_ns": tpot,
            "ttft_ok": ttft_ok, "tpot_ok": tpot_ok, "ok": ttft_ok and tpot_ok}


def attainment(records: Iterable[Dict]) -> float:
    recs = list(records)
    if not recs:
        raise ValueError("attainment of an empty run")
    return sum(1 for r in recs if r["ok"]) / len(recs)


def bisect_goodput(attain_at: Callable[[float], float], p: float, lo: float, hi: float, iters: int) -> float:
    """Largest rate in [lo, hi] with attainment >= p (attainment assumed
    non-increasing in the rate); 0 if even `lo` fails."""
    if attain_at(lo) < p:
        return 0.0
    if attain_at(hi) >= p:
        return hi
    for _ in range(iters):
        mid = 0.5 * (lo + hi)
        if attain_at(mid) >= p:
            lo = mid
        else:
            hi = mid
    return lo
