"""ORACLE (test infrastructure only) -- event-driven simulation of a PaDG macro
instance under the fixed integer cost model.

Intra-instance policy (temporal disaggregation; instance
scheduler prose P:548-553 "continues processing active decodes ... and switches
to prefills upon receiving new requests"), with the readings of DESIGN.md:
  * A15 non-preemptive: an in-flight decode step finishes before a prefill.
  * A16 a prefill window serves all pending requests FIFO in batches of at most
    `token_budget` prompt tokens (a single longer prompt forms its own batch);
    requests routed during the window join it; requests prefilled in the window
    join the decode batch when the window ends.
  * t_switch is set at every phase switch (Idle/Decode -> Prefill,
    Idle/Prefill -> Decode); A18 initial phase Idle, t_switch 0.
  * A prefill batch takes sum_r pred(S_r) ns (A13, per-request predictions
    summed); a decode step over running set R takes d + e|R| + f*sum(S+n_gen)/1000.
  * Each request's first token is stamped at the end of its prefill batch
    (n_generated = 1); every decode step adds one token; a request finishes
    when n_generated == G (A7) and frees its KV blocks.
Event order at equal time: all step completions (by instance index), then
arrivals (by request id). After every event the macro sees exact statuses
(A17), deferred requests are retried after every completion, and idle instances
are started in index order.
"""
from __future__ import annotations

import heapq
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

from .scheduler import (BLOCK_TOKENS, DEFERRED, CostModel, Macro, MacroConfig,
                        ReqStatus, ceil_div)

IDLE, PREFILL, DECODE = 0, 1, 2


@dataclass
class SimReq:
    req_id: int
    arrival_ns: int
    S: int
    G: int
    inst: int = -1
    t_first_ns: int = -1
    t_decode_begin_ns: int = -1
    t_done_ns: int = -1
    n_gen: int = 0


@dataclass
class SimInst:
    idx: int
    total_blocks: int
    phase: int = IDLE
    t_switch: int = 0
    busy: bool = False
    op: Optional[tuple] = None                      # ("prefill", [ids]) | ("decode", [ids])
    op_start: int = 0
    queue: List[int] = field(default_factory=list)  # routed, not yet prefilled (FIFO)
    waiting: List[int] = field(default_factory=list)  # prefilled in this window
    running: List[int] = field(default_factory=list)
    finished_unreported: List[int] = field(default_factory=list)
    timeline: List[tuple] = field(default_factory=list)  # (t_start, t_end, kind, n)


class Simulation:
    def __init__(self, reqs: Sequence, n_inst: int, total_blocks: int, cfg: MacroConfig,
                 cost: CostModel, token_budget: int = 16384):
        self.reqs: Dict[int, SimReq] = {r.req_id: SimReq(r.req_id, r.arrival_ns, r.prompt_len, r.output_len)
                                        for r in reqs}
        self.inst = [SimInst(i, total_blocks) for i in range(n_inst)]
        self.cost = cost
        self.budget = token_budget
        self.macro = Macro(n_inst, [total_blocks] * n_inst, cfg, cost)
        self.events: List[tuple] = []
        self.route_log: List[tuple] = []   # (t, req_id, inst or -1)
        self.max_blocks_used = [0] * n_inst

    # -------------------------------------------------------------- helpers
    @staticmethod
    def kv_len(r: SimReq) -> int:
        """Tokens whose K/V are stored: the prompt after prefill, plus one per
        completed decode step (the token fed at that step)."""
        return r.S + max(r.n_gen - 1, 0)

    def push_status(self, t: int) -> None:
        for inst in self.inst:
            reqs = []
            for rid in inst.queue + inst.waiting + inst.running + (inst.op[1] if inst.op else []):
                r = self.reqs[rid]
                reqs.append(ReqStatus(rid, r.arrival_ns, r.S, r.t_first_ns, r.n_gen, False))
            for rid in inst.finished_unreported:
                r = self.reqs[rid]
                reqs.append(ReqStatus(rid, r.arrival_ns, r.S, r.t_first_ns, r.n_gen, True))
            inst.finished_unreported.clear()
            self.macro.update_status(inst.idx, inst.phase, inst.t_switch, reqs)

    def route(self, rid: int, t: int) -> int:
        r = self.reqs[rid]
        self.push_status(t)
        i = self.macro.route(rid, r.S, r.arrival_ns, t)
        self.route_log.append((t, rid, i))
        if i != DEFERRED:
            r.inst = i
            self.inst[i].queue.append(rid)
        return i

    # -------------------------------------------------------------- policy
    def start_next(self, inst: SimInst, t: int) -> None:
        if inst.busy:
            return
        if inst.queue:
            if inst.phase != PREFILL:
                inst.phase, inst.t_switch = PREFILL, t
            batch, tok = [], 0
            while inst.queue:
                S = self.reqs[inst.queue[0]].S
                if batch and tok + S > self.budget:
                    break
                batch.append(inst.queue.pop(0))
                tok += S
            dur = sum(self.cost.prefill_ns(self.reqs[rid].S) for rid in batch)
            self.begin(inst, t, ("prefill", batch), dur)
        elif inst.waiting or inst.running:
            if inst.phase != DECODE:
                inst.phase, inst.t_switch = DECODE, t
                for rid in inst.waiting:
                    self.reqs[rid].t_decode_begin_ns = t
                inst.running.extend(inst.waiting)
                inst.waiting.clear()
            batch = list(inst.running)
            # this step appends one KV row per request: context = S + n_gen
            sum_ctx = sum(self.reqs[rid].S + self.reqs[rid].n_gen for rid in batch)
            dur = self.cost.decode_ns(len(batch), sum_ctx)
            self.begin(inst, t, ("decode", batch), dur)

    def begin(self, inst: SimInst, t: int, op: tuple, dur: int) -> None:
        inst.busy, inst.op, inst.op_start = True, op, t
        if op[0] == "decode":
            inst.running = []
        heapq.heappush(self.events, (t + dur, 0, inst.idx))

    def complete(self, inst: SimInst, t: int) -> None:
        kind, ids = inst.op
        inst.timeline.append((inst.op_start, t, kind, len(ids)))
        inst.busy, inst.op = False, None
        for rid in ids:
            r = self.reqs[rid]
            if kind == "prefill":
                r.t_first_ns, r.n_gen = t, 1
            else:
                r.n_gen += 1
            if r.n_gen >= r.G:
                r.t_done_ns = t
                if kind == "prefill":
                    r.t_decode_begin_ns = t
                inst.finished_unreported.append(rid)
            elif kind == "prefill":
                inst.waiting.append(rid)
            else:
                inst.running.append(rid)
        used = sum(ceil_div(self.kv_len(self.reqs[rid]), BLOCK_TOKENS) for rid in inst.waiting + inst.running)
        if used > inst.total_blocks:
            raise RuntimeError(f"instance {inst.idx} KV pool overflow ({used} > {inst.total_blocks}); "
                               "the reservation R is below the trace's output lengths (A14)")
        self.max_blocks_used[inst.idx] = max(self.max_blocks_used[inst.idx], used)

    # -------------------------------------------------------------- main loop
    def run(self) -> Dict[int, SimReq]:
        for rid in sorted(self.reqs):
            heapq.heappush(self.events, (self.reqs[rid].arrival_ns, 1, rid))
        while self.events:
            t, kind, idx = heapq.heappop(self.events)
            if kind == 0:
                self.complete(self.inst[idx], t)
                self.push_status(t)
                for rid, i in self.macro.drain_deferred(t):
                    self.reqs[rid].inst = i
                    self.inst[i].queue.append(rid)
                    self.route_log.append((t, rid, i))
            else:
                if self.route(idx, t) == DEFERRED:
                    r = self.reqs[idx]
                    self.macro.deferred.append((idx, r.S, r.arrival_ns))
            for inst in self.inst:
                self.start_next(inst, t)
        return self.reqs


def simulate(reqs, n_inst: int, total_blocks: int, cfg: MacroConfig, cost: CostModel,
             token_budget: int = 16384) -> Simulation:
    sim = Simulation(reqs, n_inst, total_blocks, cfg, cost, token_budget)
    sim.run()
    return sim
