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
  * A14 KV pressure (only when the reservation R is below a request's true
    output, so C3 admitted more than the pool holds): a decode step first checks
    that every request of its batch can hold ceil((S + n_gen)/64) blocks after
    the step; while it cannot, the latest-arrived request of the batch (largest
    (arrival, id)) is preempted -- its blocks are freed and it goes to the FRONT
    of the instance's queue as a recompute: a prefill of its prompt plus all
    n_gen generated tokens (TD-Pipe's recompute), which yields its next
    token (n_gen + 1; t_first and t_decode_begin keep their first values).
    A prefill batch is the FIFO prefix of the queue that fits both the token
    budget and the free blocks; when the head does not fit, the instance keeps
    decoding until completions free enough blocks.
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
    n_preempt: int = 0   # times preempted for recompute (A14)


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
        self.preempt_log: List[tuple] = []  # (t, req_id, inst) of every A14 preemption

    # -------------------------------------------------------------- helpers
    @staticmethod
    def kv_len(r: SimReq) -> int:
        """Tokens whose K/V are stored: the prompt after prefill, plus one per
        completed decode step (the token fed at that step)."""
        return r.S + max(r.n_gen - 1, 0)

    @staticmethod
    def prefill_len(r: SimReq) -> int:
        """Tokens a prefill of r processes: its prompt, or for a recompute after a
        preemption (A14) the prompt plus every generated token."""
        return r.S + r.n_gen

    def held_blocks(self, inst: SimInst) -> int:
        return sum(ceil_div(self.kv_len(self.reqs[rid]), BLOCK_TOKENS) for rid in inst.waiting + inst.running)

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
        free = inst.total_blocks - self.held_blocks(inst)
        head = self.reqs[inst.queue[0]] if inst.queue else None
        if head is not None and ceil_div(self.prefill_len(head), BLOCK_TOKENS) <= free:
            if inst.phase != PREFILL:
                inst.phase, inst.t_switch = PREFILL, t
            batch, tok = [], 0
            while inst.queue:
                r = self.reqs[inst.queue[0]]
                n_tok, need = self.prefill_len(r), ceil_div(self.prefill_len(r), BLOCK_TOKENS)
                if batch and tok + n_tok > self.budget:
                    break
                if need > free:
                    break
                batch.append(inst.queue.pop(0))
                tok += n_tok
                free -= need
            dur = sum(self.cost.prefill_ns(self.prefill_len(self.reqs[rid])) for rid in batch)
            self.begin(inst, t, ("prefill", batch), dur)
        elif inst.waiting or inst.running:
            if inst.phase != DECODE:
                inst.phase, inst.t_switch = DECODE, t
                for rid in inst.waiting:
                    if self.reqs[rid].t_decode_begin_ns < 0:
                        self.reqs[rid].t_decode_begin_ns = t
                inst.running.extend(inst.waiting)
                inst.waiting.clear()
            batch = list(inst.running)
            # A14: after this step request b holds ceil((S + n_gen)/64) blocks; preempt the
            # latest arrival until the batch fits (front of the queue, FIFO among them)
            while batch and sum(ceil_div(self.reqs[rid].S + self.reqs[rid].n_gen, BLOCK_TOKENS)
                                for rid in batch) > inst.total_blocks:
                v = max(batch, key=lambda rid: (self.reqs[rid].arrival_ns, rid))
                batch.remove(v)
                inst.running.remove(v)
                inst.queue.insert(0, v)
                self.reqs[v].n_preempt += 1
                self.preempt_log.append((t, v, inst.idx))
            if not batch:
                raise RuntimeError(f"instance {inst.idx}: one request outgrew the whole KV pool")
            # this step appends one KV row per request: context = S + n_gen
            sum_ctx = sum(self.reqs[rid].S + self.reqs[rid].n_gen for rid in batch)
            dur = self.cost.decode_ns(len(batch), sum_ctx)
            self.begin(inst, t, ("decode", batch), dur)
        elif head is not None:
            raise RuntimeError(f"instance {inst.idx}: request {head.req_id} needs more blocks than the pool holds")

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
            if kind == "prefill" and r.n_gen == 0:
                r.t_first_ns, r.n_gen = t, 1
            else:  # a decode step, or a recompute prefill (A14): the next token
                r.n_gen += 1
            if r.n_gen >= r.G:
                r.t_done_ns = t
                if kind == "prefill" and r.t_decode_begin_ns < 0:
                    r.t_decode_begin_ns = t
                inst.finished_unreported.append(rid)
            elif kind == "prefill":
                inst.waiting.append(rid)
            else:
                inst.running.append(rid)
        used = self.held_blocks(inst)
        if used > inst.total_blocks:  # invariant: the A14 admission / preemption rule prevents it
            raise RuntimeError(f"instance {inst.idx} KV pool overflow ({used} > {inst.total_blocks})")
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
