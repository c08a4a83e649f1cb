"""Live PaDG serving of one macro instance over real GPU instances
(SURVEY 8(a) rows a1-a4 and a18 in live mode).

* One worker thread per GPU instance runs the intra-instance policy (temporal
  disaggregation): after every decode step, if the
  macro forwarded requests, it switches to a prefill phase that drains them FIFO
  in <= token_budget batches (A16), then switches back to decode; it stamps
  t_first / t_decode_begin / t_done with the host clock and pushes its status
  (decode progress, memory use) to the macro after every phase call.
* The dispatcher thread replays the trace in real time (Poisson arrivals)
  and routes every arrival with the C++ macro scheduler (Alg. 1/2),
  deferring when no instance passes CheckConstraints; rolling activation
  emerges from the routing.
* Metrics per Sec. 3.3: reported TTFT includes the phase-switch
  wait; TPOT is measured from the first decode step after the switch.

The ctypes calls into libecoserve.so release the GIL, so N instances on N GPUs
run concurrently from one process.

policy="nodg" is the paper's NoDG separate-batching baseline (vLLM-style,
P:312-320, 675-676) on the same kernels and the same per-instance
prefill-priority loop: every arrival is routed immediately, round-robin, with no
constraint check and no deferral, so every instance interleaves prefills into
its decode stream (no rolling activation).

policy="fudg" is the fully disaggregated baseline (DistServe-style FuDG, P:321-354;
SURVEY 8(f) N4(i)) on the same kernels: the first `fudg_prefill` instances only
prefill (arrivals round-robin over them), every prefilled request's paged KV is
exported over NVLink into a staging buffer on a decode instance (round-robin over
the others), which imports it on its own thread and only decodes. The KV transfer
the paper's PaDG avoids is on the critical path between the first token and the
first decode step (it counts as switch wait).

policy="sarathi" is the NoDG hybrid-batching baseline (Sarathi-Serve):
round-robin routing, and every worker iteration is ONE forward pass
(Instance.hybrid_step) that decodes every running request by one token and fills
the rest of a per-iteration token budget (`chunk_budget`) with prompt chunks,
FIFO; a request starts decoding in the iteration after its last chunk.
"""
from __future__ import annotations

import queue
import threading
import time
from collections import deque
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np

from .macro import MacroScheduler, SchedConfig

IDLE, PREFILL, DECODE = 0, 1, 2
FUDG_BACKLOG = 64  # staged (exported, not yet imported) requests per FuDG decode instance


@dataclass
class LiveReq:
    req_id: int
    arrival_ns: int
    prompt: np.ndarray
    G: int
    inst: int = -1
    t_first_ns: int = -1
    t_decode_begin_ns: int = -1
    t_done_ns: int = -1
    n_gen: int = 0
    tokens: List[int] = field(default_factory=list)

    @property
    def S(self) -> int:
        return len(self.prompt)


class Clock:
    def __init__(self):
        self.t0 = time.perf_counter_ns()

    def now(self) -> int:
        return time.perf_counter_ns() - self.t0


class Worker(threading.Thread):
    def __init__(self, idx: int, inst, clock: Clock, status_q: "queue.Queue", token_budget: int,
                 decode_steps_per_poll: int = 1, max_batch: int = 256, hybrid_budget: int = 0,
                 role: str = "both", handoff=None, admission: str = "reserve"):
        super().__init__(daemon=True)
        # "reserve": FCFS reservation of prompt + output blocks (no preemption ever needed);
        # "preempt": reading A14 -- admit on the prompt's blocks, and before a decode step that
        # would outgrow the pool preempt the latest arrivals for recompute (as oracle/des.py)
        if admission not in ("reserve", "preempt"):
            raise ValueError(f"unknown admission {admission!r}")
        self.admission = admission
        self.n_preempted = 0
        self.hybrid_budget = hybrid_budget   # > 0: Sarathi-style hybrid iterations
        self.role = role                     # "both" | "prefill" | "decode" (FuDG)
        self.handoff = handoff               # FuDG prefill role: () -> the decode Worker for the next request
        self.imports: deque = deque()        # FuDG decode role: (req, kv handle) waiting for blocks
        self.decode_full = lambda: False     # FuDG prefill role: set by the server
        self.idx, self.inst, self.clock = idx, inst, clock
        self.inbox: "queue.Queue" = queue.Queue()
        self.status_q = status_q
        self.budget = token_budget
        self.k = decode_steps_per_poll
        self.max_batch = max_batch
        self.stop_flag = threading.Event()
        self.phase, self.t_switch = IDLE, 0
        self.pending: deque = deque()
        self.waiting: List[LiveReq] = []
        self.running: List[LiveReq] = []
        self.finished: List[LiveReq] = []
        self.timeline: List[tuple] = []
        self.error: Optional[BaseException] = None
        # KV admission control (FCFS): a request starts its prefill only when the blocks
        # its prompt + output can reach fit next to those committed to live requests
        # (there is no preemption, reading A14), so no policy can exhaust the pool
        self.total_blocks = int(getattr(inst, "num_blocks", 1 << 30))
        self.committed: Dict[int, int] = {}
        self.commit_sum = 0
        # mitosis (N1, live): a contracted instance drains -- every prefilled request moves
        # with its paged KV (export_kv / import_kv over NVLink) to drain_dst(), pending ones
        # are re-queued there -- and then idles until the macro grows again
        self.draining = False
        self.drain_dst = None
        self.n_migrated_out = 0
        self.migrate_ns = 0

    def _fits(self, r: LiveReq, extra: int = 0) -> bool:
        if self.admission == "preempt":  # the prompt (plus regenerated tokens) must fit now
            return self._held() + extra + (r.S + r.n_gen + 63) // 64 <= self.total_blocks
        return r.req_id in self.committed or \
            self.commit_sum + (r.S + r.G + 63) // 64 <= self.total_blocks

    def _held(self) -> int:
        """Blocks the engine holds for prefilled requests: prompt + fed tokens (A14)."""
        return sum((r.S + r.n_gen - 1 + 63) // 64 for r in self.waiting + self.running)

    def _preempt_for(self, steps: int) -> None:
        """Reading A14 in live mode: while the running batch would need more blocks than the
        pool after `steps` decode steps, release the latest-arrived request and put it at the
        front of the queue; its recompute prefill feeds prompt + every generated token."""
        def need():
            return sum((r.S + min(r.n_gen + steps, r.G) - 1 + 63) // 64 for r in self.running)
        while len(self.running) > 1 and need() > self.total_blocks:
            v = max(self.running, key=lambda r: (r.arrival_ns, r.req_id))
            self.running.remove(v)
            self.inst.release([v.req_id])
            self.pending.appendleft(v)
            self.n_preempted += 1

    def _commit(self, r: LiveReq) -> None:
        if r.req_id not in self.committed:
            need = (r.S + r.G + 63) // 64
            self.committed[r.req_id] = need
            self.commit_sum += need

    def push_status(self, fin: Sequence[LiveReq] = ()):
        live = list(self.pending) + self.waiting + self.running
        if self.role == "both":  # requests migrated here whose KV is not imported yet
            live += [r for r, _ in self.imports]
        recs = [(r.req_id, r.arrival_ns, r.S, r.t_first_ns, r.n_gen, False) for r in live]
        recs += [(r.req_id, r.arrival_ns, r.S, r.t_first_ns, r.n_gen, True) for r in fin]
        self.status_q.put((self.idx, self.phase, self.t_switch, recs))

    def _take(self, item) -> None:
        if isinstance(item, tuple) and item[0] == "import":  # a migrated request and its staged KV
            self.imports.append((item[1], item[2]))
        elif isinstance(item, tuple) and item[0] == "drain":
            self.draining = True
        elif isinstance(item, tuple) and item[0] == "requeue":  # from a drained instance: arrival order
            r, i = item[1], len(self.pending)
            while i > 0 and self.pending[i - 1].arrival_ns > r.arrival_ns:
                i -= 1
            self.pending.insert(i, r)
        else:
            self.pending.append(item)

    def _drain_inbox(self, block: bool):
        try:
            self._take(self.inbox.get(timeout=0.002) if block else self.inbox.get_nowait())
            while True:
                self._take(self.inbox.get_nowait())
        except queue.Empty:
            pass

    def _drain_out(self) -> None:
        """Mitosis contraction: hand every request of this instance to the
        remaining ones -- prefilled requests with their KV blocks (NVLink peer copy into a
        staging buffer on the destination GPU, imported by the destination's own worker),
        queued ones as plain arrivals -- and leave the instance empty."""
        t0 = time.perf_counter_ns()
        for r in self.waiting + self.running:
            dst = self.drain_dst()
            handle = self.inst.export_kv(r.req_id, dst.inst.device)
            self.commit_sum -= self.committed.pop(r.req_id, 0)
            r.inst = dst.idx
            dst.inbox.put(("import", r, handle))
            self.n_migrated_out += 1
        for r, handle in list(self.imports):  # in transit through this instance: forward
            dst = self.drain_dst()
            r.inst = dst.idx
            dst.inbox.put(("import", r, handle))
        while self.pending:
            r = self.pending.popleft()
            self.commit_sum -= self.committed.pop(r.req_id, 0)
            dst = self.drain_dst()
            r.inst = dst.idx
            dst.inbox.put(("requeue", r))
        self.waiting, self.running = [], []
        self.imports.clear()
        self.migrate_ns += time.perf_counter_ns() - t0
        self.draining = False
        self.phase, self.t_switch = IDLE, self.clock.now()
        self.push_status()

    def _admit_imports(self) -> None:
        """Migrated requests join this instance's decode set once their blocks fit."""
        while self.imports and self._fits(self.imports[0][0]):
            r, handle = self.imports.popleft()
            self.inst.import_kv(handle)
            self._commit(r)
            if self.phase == DECODE:  # joins the running decode set now
                if r.t_decode_begin_ns < 0:
                    r.t_decode_begin_ns = self.clock.now()
                self.running.append(r)
            else:  # joins at this instance's next switch to decode
                self.waiting.append(r)

    def run(self):
        try:
            if self.hybrid_budget > 0:
                self._loop_hybrid()
            elif self.role == "decode":
                self._loop_decode_only()
            else:
                self._loop()
        except BaseException as e:  # surfaced by the server
            self.error = e

    def _loop_hybrid(self):
        """Sarathi-style stall-free batching: every iteration decodes all running
        requests by one token and spends the rest of the token budget on prompt chunks."""
        prefilled: Dict[int, int] = {}
        self.phase = DECODE
        while not self.stop_flag.is_set():
            self._drain_inbox(block=False)
            if not self.running and (not self.pending or not self._fits(self.pending[0])):
                self._drain_inbox(block=True)
                continue
            dec = list(self.running)
            budget = self.hybrid_budget - len(dec)
            chunks, taken = [], []
            for r in self.pending:
                if budget <= 0 or len(chunks) + len(dec) >= self.max_batch or not self._fits(r):
                    break
                self._commit(r)
                done = prefilled.get(r.req_id, 0)
                take = min(budget, r.S - done)
                chunks.append((r.req_id, r.prompt, r.G, take))
                taken.append((r, take))
                budget -= take
            t0 = self.clock.now()
            ct, dt = self.inst.hybrid_step(chunks, [r.req_id for r in dec])
            t = self.clock.now()
            self.timeline.append((t0, t, "hybrid", len(dec), sum(x[1] for x in taken)))
            fin, keep = [], []
            for r, tok in zip(dec, dt):
                r.tokens.append(int(tok))
                r.n_gen += 1
                if r.n_gen >= r.G:
                    r.t_done_ns = t
                    fin.append(r)
                else:
                    keep.append(r)
            for (r, take), tok in zip(taken, ct):
                prefilled[r.req_id] = prefilled.get(r.req_id, 0) + take
                if tok >= 0:  # the prompt is complete: first token
                    self.pending.remove(r)
                    prefilled.pop(r.req_id, None)
                    r.t_first_ns = r.t_decode_begin_ns = t
                    r.n_gen = 1
                    r.tokens.append(int(tok))
                    if r.G <= 1:
                        r.t_done_ns = t
                        fin.append(r)
                    else:
                        keep.append(r)
            self.running = keep
            self._finish(fin)
            self.push_status(fin)

    def backlog(self) -> int:
        """FuDG decode role: handed-off requests not yet imported (their KV sits in staging)."""
        return len(self.imports) + self.inbox.qsize()

    def _loop(self):
        while not self.stop_flag.is_set():
            self._drain_inbox(block=False)
            if self.draining:
                self._drain_out()
                continue
            if self.imports:
                self._admit_imports()
            if self.role == "prefill" and self.decode_full():
                # back-pressure: the decode instances have FUDG_BACKLOG staged requests each
                # (their KV waits in staging buffers on the decode GPUs); prefill again later
                self._drain_inbox(block=True)
                continue
            if self.pending and self._fits(self.pending[0]):
                if self.phase != PREFILL:
                    self.phase, self.t_switch = PREFILL, self.clock.now()
                batch, tok, extra = [], 0, 0
                while self.pending and len(batch) < self.max_batch and \
                        (not batch or tok + self.pending[0].S + self.pending[0].n_gen <= self.budget) and \
                        self._fits(self.pending[0], extra):
                    r = self.pending.popleft()
                    self._commit(r)
                    batch.append(r)
                    tok += r.S + r.n_gen
                    extra += (r.S + r.n_gen + 63) // 64  # (preempt admission: blocks of this batch)
                t0 = self.clock.now()
                # a recompute (A14) prefills the prompt and every generated token; the engine
                # request then owes the remaining G - n_gen tokens
                first = self.inst.prefill([(r.req_id, self._prefill_ids(r), r.G - r.n_gen) for r in batch])
                t = self.clock.now()
                self.timeline.append((t0, t, "prefill", len(batch)))
                fin = []
                for r, f in zip(batch, first):
                    if r.n_gen == 0:
                        r.t_first_ns = t
                    r.n_gen += 1
                    r.tokens.append(int(f))
                    if r.n_gen >= r.G:
                        if r.t_decode_begin_ns < 0:
                            r.t_decode_begin_ns = t
                        r.t_done_ns = t
                        fin.append(r)
                    elif self.role == "prefill":  # FuDG: the KV moves to a decode instance
                        dst = self.handoff()
                        handle = self.inst.export_kv(r.req_id, dst.inst.device)
                        self.commit_sum -= self.committed.pop(r.req_id, 0)
                        dst.inbox.put((r, handle))
                    else:
                        self.waiting.append(r)
                self._finish(fin)
                self.push_status(fin)
            elif self.waiting or self.running:
                if self.phase != DECODE:
                    self.phase, self.t_switch = DECODE, self.clock.now()
                    for r in self.waiting:
                        if r.t_decode_begin_ns < 0:
                            r.t_decode_begin_ns = self.t_switch
                    self.running += self.waiting
                    self.waiting = []
                if self.admission == "preempt":
                    self._preempt_for(self.k)
                t0 = self.clock.now()
                ids = [r.req_id for r in self.running]
                # decode phases of <= max_batch requests (the instance's batch limit)
                parts = [self.inst.decode(ids[i:i + self.max_batch], self.k)[0]
                         for i in range(0, len(ids), self.max_batch)]
                toks = np.concatenate(parts, axis=0) if parts else np.zeros((0, self.k), np.int32)
                t = self.clock.now()
                self.timeline.append((t0, t, "decode", len(self.running)))
                fin, keep = [], []
                for i, r in enumerate(self.running):
                    for s in range(self.k):
                        if toks[i, s] >= 0:
                            r.tokens.append(int(toks[i, s]))
                            r.n_gen += 1
                    if r.n_gen >= r.G:
                        r.t_done_ns = t
                        fin.append(r)
                    else:
                        keep.append(r)
                self.running = keep
                self._finish(fin)
                self.push_status(fin)
            else:
                self._drain_inbox(block=True)

    def _loop_decode_only(self):
        """FuDG decode instance: imports handed-off requests (KV already prefilled on a
        prefill instance) as blocks allow, and runs decode steps over its running set."""
        self.phase = DECODE
        while not self.stop_flag.is_set():
            try:
                while True:
                    self.imports.append(self.inbox.get_nowait())
            except queue.Empty:
                pass
            while self.imports and len(self.running) < self.max_batch and self._fits(self.imports[0][0]):
                r, handle = self.imports.popleft()
                self.inst.import_kv(handle)
                self._commit(r)
                r.t_decode_begin_ns = self.clock.now()
                self.running.append(r)
            if not self.running:
                try:
                    self.imports.append(self.inbox.get(timeout=0.002))
                except queue.Empty:
                    pass
                continue
            t0 = self.clock.now()
            toks, _ = self.inst.decode([r.req_id for r in self.running], self.k)
            t = self.clock.now()
            self.timeline.append((t0, t, "decode", len(self.running)))
            fin, keep = [], []
            for i, r in enumerate(self.running):
                for s_ in range(self.k):
                    if toks[i, s_] >= 0:
                        r.tokens.append(int(toks[i, s_]))
                        r.n_gen += 1
                if r.n_gen >= r.G:
                    r.t_done_ns = t
                    fin.append(r)
                else:
                    keep.append(r)
            self.running = keep
            self._finish(fin)
            self.push_status(fin)

    @staticmethod
    def _prefill_ids(r: LiveReq) -> np.ndarray:
        if r.n_gen == 0:
            return r.prompt
        return np.concatenate([r.prompt, np.asarray(r.tokens, dtype=np.int32)])

    def _finish(self, fin):
        if fin:
            self.inst.release([r.req_id for r in fin])
            self.finished += fin
            for r in fin:
                self.commit_sum -= self.committed.pop(r.req_id, 0)


def profile_prefill(inst, lens=(128, 256, 512, 1024, 2048, 4096), vocab: int = 1000, reps: int = 2):
    """On-box prefill profile (P:513 'predicted in advance by profiling sequences
    of various lengths'; reading A13): median ns of a single-request prefill phase."""
    rng = np.random.default_rng(0)
    out_l, out_ns = [], []
    rid = -1_000_000
    for S in lens:
        ts = []
        for _ in range(reps + 1):
            p = rng.integers(0, vocab, S).astype(np.int32)
            t0 = time.perf_counter_ns()
            inst.prefill([(rid, p, 1)])
            ts.append(time.perf_counter_ns() - t0)
            inst.release([rid])
            rid -= 1
        out_l.append(S)
        out_ns.append(int(np.median(ts[1:])))
    return out_l, out_ns


class PaDGServer:
    """A macro instance of len(instances) GPU instances under rolling activation."""

    def __init__(self, instances: Sequence, slo_ttft_ns: int, slo_tpot_ns: int, reserve_tokens: int,
                 predictor_table=None, token_budget: int = 16384, decode_steps_per_poll: int = 1,
                 probe_printed: bool = False, policy: str = "padg", chunk_budget: int = 1024,
                 fudg_prefill: int = 0, admission: str = "reserve", resize=None):
        """resize (mitosis, N1 live; padg only): [(t_s, n_active), ...] -- from t_s seconds
        into the run the macro holds instances [0, n_active): expansion activates the next
        instances (the router starts probing them), contraction drains the highest ones into
        the remaining (running requests move with their KV over NVLink). Before the first
        event all instances are active unless the first event is at t_s = 0. A dict
        ({n_min, n_max, n_start, up_s, down_s, down_live, cooldown_s}) selects the automatic
        triggers of _auto_resize instead."""
        if policy not in ("padg", "nodg", "sarathi", "fudg"):
            raise ValueError(f"unknown policy {policy!r}")
        if isinstance(resize, dict):  # automatic triggers, see _auto_resize
            self.auto = dict(n_min=1, n_max=len(instances), up_s=0.5, down_s=10.0, down_live=2, cooldown_s=5.0)
            self.auto.update(resize)
            resize = [(0, self.auto.pop("n_start", self.auto["n_min"]))]
        else:
            self.auto = None
        if resize and policy != "padg":
            raise ValueError("live mitosis (resize) is implemented for the padg policy")
        if resize and not all(hasattr(i, "export_kv") and hasattr(i, "import_kv") for i in instances):
            raise ValueError("live mitosis moves KV: every instance needs export_kv / import_kv (TP=1)")
        self.resize = sorted(resize or [])
        self.n_active = len(instances)
        self.resize_log: List[tuple] = []
        self.n_deferred = 0
        self.policy = policy
        self._rr = 0
        self.clock = Clock()
        self.status_q: "queue.Queue" = queue.Queue()
        hb = chunk_budget if policy == "sarathi" else 0
        n = len(instances)
        self.n_prefill = n
        roles = ["both"] * n
        if policy == "fudg":
            if n < 2:
                raise ValueError("fudg needs >= 2 instances (prefill and decode roles)")
            self.n_prefill = fudg_prefill if 0 < fudg_prefill < n else n // 2
            roles = ["prefill"] * self.n_prefill + ["decode"] * (n - self.n_prefill)
        self._rr_dec = 0
        self._rr_lock = threading.Lock()  # several prefill workers hand off concurrently

        def handoff():
            dec = self.workers[self.n_prefill:]
            with self._rr_lock:
                w = dec[self._rr_dec % len(dec)]
                self._rr_dec += 1
            return w

        if admission == "preempt" and policy not in ("padg", "nodg"):
            raise ValueError("preempt admission is implemented for the separate-batching loops (padg, nodg)")
        self.workers = [Worker(i, inst, self.clock, self.status_q, token_budget, decode_steps_per_poll,
                               hybrid_budget=hb, role=roles[i], handoff=handoff, admission=admission)
                        for i, inst in enumerate(instances)]
        if policy == "fudg":
            def decode_full():
                dec = self.workers[self.n_prefill:]
                return sum(w.backlog() for w in dec) >= FUDG_BACKLOG * len(dec)
            for w in self.workers[:self.n_prefill]:
                w.decode_full = decode_full
        blocks = [inst.num_blocks for inst in instances]
        self.macro = MacroScheduler(SchedConfig(len(instances), slo_ttft_ns, slo_tpot_ns, reserve_tokens, blocks,
                                                probe_printed=probe_printed, table=predictor_table))
        self.route_log: List[tuple] = []
        self.reqs: Dict[int, LiveReq] = {}

    def _apply_statuses(self):
        n = 0
        while True:
            try:
                idx, phase, t_switch, recs = self.status_q.get_nowait()
            except queue.Empty:
                break
            self.macro.update_status(idx, phase, t_switch, self.workers[idx].inst.num_blocks, recs,
                                     alive=idx < self.n_active)
            n += 1
        if n:
            for rid, i in self.macro.drain_deferred(self.clock.now()):
                self.n_deferred -= 1
                self._send(self.reqs[rid], i)

    def _apply_resize(self, n_new: int) -> None:
        """Mitosis step: grow or shrink the active prefix of the macro to n_new instances."""
        n_new = max(1, min(n_new, len(self.workers)))
        n_old, self.n_active = self.n_active, n_new
        self.resize_log.append((self.clock.now(), n_old, n_new))
        for idx in range(min(n_old, n_new), max(n_old, n_new)):
            w = self.workers[idx]
            if n_new < n_old:  # contraction: drain into the least-loaded remaining instance
                keep = self.workers[:n_new]

                def dst(keep=keep):
                    return min(keep, key=lambda k: (len(k.pending) + len(k.waiting) + len(k.running) +
                                                    len(k.imports) + k.inbox.qsize(), k.idx))
                w.drain_dst = dst
                w.inbox.put(("drain",))
            # the router's view: alive only inside the active prefix (expansion: empty status)
            self.macro.update_status(idx, w.phase, w.t_switch, w.inst.num_blocks, [], alive=idx < n_new)

    def _auto_resize(self, now: int) -> None:
        """Mitosis triggers (scale "when the system fails to meet the defined SLOs or
        when there is sustained resource underutilization"): expand by one instance once
        requests have stayed Deferred -- no active instance passes Alg. 2 -- for up_s seconds;
        contract by one once nothing was deferred for down_s seconds and the last active
        instance holds <= down_live live requests (they move with their KV). One step per
        cooldown_s."""
        a = self.auto
        if now - self._auto_last < a["cooldown_s"] * 1e9:
            return
        if self.n_deferred > 0:
            self._auto_quiet = now
            if self._auto_busy < 0:
                self._auto_busy = now
            if now - self._auto_busy >= a["up_s"] * 1e9 and self.n_active < a["n_max"]:
                self._apply_resize(self.n_active + 1)
                self._auto_last, self._auto_busy = now, -1
            return
        self._auto_busy = -1
        w = self.workers[self.n_active - 1]
        live = len(w.pending) + len(w.waiting) + len(w.running) + len(w.imports)
        if (now - self._auto_quiet >= a["down_s"] * 1e9 and self.n_active > a["n_min"] and
                live <= a["down_live"]):
            self._apply_resize(self.n_active - 1)
            self._auto_last, self._auto_quiet = now, now

    def _send(self, r: LiveReq, i: int):
        r.inst = i
        self.route_log.append((self.clock.now(), r.req_id, i))
        self.workers[i].inbox.put(r)

    def run(self, trace, timeout_s: float = 600.0) -> Dict[int, LiveReq]:
        """Replay `trace` (synthetic.traces.Request with prompts) in real time."""
        for w in self.workers:
            w.start()
        reqs = sorted(trace, key=lambda r: (r.arrival_ns, r.req_id))
        t_start = self.clock.now()
        for r in reqs:
            lr = LiveReq(r.req_id, t_start + r.arrival_ns, np.asarray(r.prompt, np.int32), r.output_len)
            self.reqs[r.req_id] = lr
        pending = deque(self.reqs[r.req_id] for r in reqs)
        events = deque(self.resize)
        if events and events[0][0] <= 0:
            self._apply_resize(events.popleft()[1])
        self._auto_last = self._auto_quiet = t_start
        self._auto_busy = -1
        deadline = time.perf_counter() + timeout_s
        while time.perf_counter() < deadline:
            self._apply_statuses()
            now = self.clock.now()
            while events and now - t_start >= events[0][0] * 1e9:
                self._apply_resize(events.popleft()[1])
            if self.auto is not None:
                self._auto_resize(now)
            while pending and pending[0].arrival_ns <= now:
                lr = pending.popleft()
                if self.policy != "padg":  # immediate round-robin dispatch (NoDG / FuDG prefill instances)
                    i, self._rr = self._rr, (self._rr + 1) % self.n_prefill
                    self._send(lr, i)
                    continue
                i, _ = self.macro.route(lr.req_id, lr.arrival_ns, lr.S, now)
                if i < 0:
                    self.route_log.append((now, lr.req_id, -1))
                    self.macro.defer(lr.req_id, lr.arrival_ns, lr.S)
                    self.n_deferred += 1
                else:
                    self._send(lr, i)
            for w in self.workers:
                if w.error is not None:
                    raise RuntimeError(f"instance {w.idx} failed") from w.error
            if not pending and all(r.t_done_ns >= 0 for r in self.reqs.values()):
                break
            time.sleep(0.0005)
        for w in self.workers:
            w.stop_flag.set()
        for w in self.workers:
            w.join(timeout=30)
        self._release_leftovers()
        return self.reqs

    def _release_leftovers(self):
        """A run that stops early (timeout, worker error) leaves requests resident:
        unfinished decodes, partly chunked prompts, FuDG requests exported but never
        imported. Release them and drop staged KV handles so the instances (reused by
        the next goodput probe) start from an empty pool."""
        for w in self.workers:
            if w.is_alive():
                continue  # still inside a phase call; the instance is not safe to touch
            w.imports.clear()
            while True:
                try:
                    w.inbox.get_nowait()
                except queue.Empty:
                    break
            try:
                st, recs = w.inst.status()
            except Exception:  # a dead instance: nothing to release
                continue
            if recs:
                w.inst.release([r["req_id"] for r in recs])
            w.committed.clear()
            w.commit_sum = 0
