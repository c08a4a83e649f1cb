"""ORACLE pin (test infrastructure only) -- a naive fixed-tick simulator of the
same PaDG semantics as ``des.py`` (SURVEY 8(c) "Phase timeline: event-driven DES
== naive tick simulator on tiny traces, bit-exact").

No event queue: time advances one tick at a time; at each tick every instance
whose operation ends now completes (index order, each followed by a deferred
retry), then every request arriving now is routed (id order); after each of
those, idle instances are started. Written independently of des.py: it keeps
its own per-request arrays and scans them; it shares only the Alg. 1/2 code
(scheduler.Macro) whose decisions it exercises. All durations and arrival
times must be multiples of `tick`.
"""
from __future__ import annotations

from typing import List

from .scheduler import DEFERRED, Macro, ReqStatus


def tick_simulate(reqs, n_inst: int, total_blocks: int, cfg, cost, token_budget: int, tick: int,
                  horizon: int):
    n = len(reqs)
    ids = [r.req_id for r in reqs]
    pos = {rid: k for k, rid in enumerate(ids)}
    arr = [r.arrival_ns for r in reqs]
    S = [r.prompt_len for r in reqs]
    G = [r.output_len for r in reqs]
    first = [-1] * n
    dbeg = [-1] * n
    done = [-1] * n
    ngen = [0] * n
    where = [-1] * n
    preempts = []                # (t, req_id, inst): A14 recompute preemptions
    # per instance
    phase = [0] * n_inst
    tsw = [0] * n_inst
    end = [-1] * n_inst          # end time of the in-flight op, -1 = free
    opkind = [None] * n_inst
    opids: List[List[int]] = [[] for _ in range(n_inst)]
    queue: List[List[int]] = [[] for _ in range(n_inst)]
    waiting: List[List[int]] = [[] for _ in range(n_inst)]
    running: List[List[int]] = [[] for _ in range(n_inst)]
    fin_unrep: List[List[int]] = [[] for _ in range(n_inst)]
    macro = Macro(n_inst, [total_blocks] * n_inst, cfg, cost)
    deferred: List[int] = []
    log = []

    def push():
        for i in range(n_inst):
            rs = [ReqStatus(ids[k], arr[k], S[k], first[k], ngen[k], False)
                  for k in queue[i] + waiting[i] + running[i] + opids[i]]
            rs += [ReqStatus(ids[k], arr[k], S[k], first[k], ngen[k], True) for k in fin_unrep[i]]
            fin_unrep[i] = []
            macro.update_status(i, phase[i], tsw[i], rs)

    def blocks(tokens):          # 64-token KV blocks holding `tokens` tokens
        return -(-tokens // 64)

    def kick(t):
        for i in range(n_inst):
            if end[i] >= 0:
                continue
            # blocks held: prompt + fed tokens of every prefilled request on the instance
            held = 0
            for k in waiting[i] + running[i]:
                held += blocks(S[k] + ngen[k] - 1)
            # a prefill processes the prompt, plus the generated tokens after a preemption
            if queue[i] and blocks(S[queue[i][0]] + ngen[queue[i][0]]) + held <= total_blocks:
                if phase[i] != 1:
                    phase[i], tsw[i] = 1, t
                batch, tok = [], 0
                while queue[i]:
                    k = queue[i][0]
                    if batch and tok + S[k] + ngen[k] > token_budget:
                        break
                    if held + blocks(S[k] + ngen[k]) > total_blocks:
                        break
                    queue[i].pop(0)
                    batch.append(k)
                    tok += S[k] + ngen[k]
                    held += blocks(S[k] + ngen[k])
                d = 0
                for k in batch:
                    d += cost.prefill_ns(S[k] + ngen[k])
                if d % tick:
                    raise ValueError("prefill duration is not a multiple of the tick")
                end[i], opkind[i], opids[i] = t + d, "prefill", batch
            elif waiting[i] or running[i]:
                if phase[i] != 2:
                    phase[i], tsw[i] = 2, t
                    for k in waiting[i]:
                        if dbeg[k] == -1:
                            dbeg[k] = t
                    running[i] = running[i] + waiting[i]
                    waiting[i] = []
                batch = running[i]
                running[i] = []
                # every member grows to S + ngen tokens in this step; drop latest arrivals
                # to the queue front until that fits (A14)
                while batch:
                    after = 0
                    for k in batch:
                        after += blocks(S[k] + ngen[k])
                    if after <= total_blocks:
                        break
                    late = batch[0]
                    for k in batch:
                        if (arr[k], ids[k]) > (arr[late], ids[late]):
                            late = k
                    batch.remove(late)
                    queue[i].insert(0, late)
                    preempts.append((t, ids[late], i))
                d = cost.decode_ns(len(batch), sum(S[k] + ngen[k] for k in batch))
                if d % tick:
                    raise ValueError("decode duration is not a multiple of the tick")
                end[i], opkind[i], opids[i] = t + d, "decode", batch

    t = 0
    while t <= horizon:
        for i in range(n_inst):
            if end[i] == t:
                for k in opids[i]:
                    if opkind[i] == "prefill" and first[k] == -1:
                        first[k], ngen[k] = t, 1
                    else:
                        ngen[k] += 1
                    if ngen[k] >= G[k]:
                        done[k] = t
                        if opkind[i] == "prefill" and dbeg[k] == -1:
                            dbeg[k] = t
                        fin_unrep[i].append(k)
                    elif opkind[i] == "prefill":
                        waiting[i].append(k)
                    else:
                        running[i].append(k)
                end[i], opkind[i], opids[i] = -1, None, []
                push()
                while deferred:
                    k = deferred[0]
                    j = macro.route(ids[k], S[k], arr[k], t)
                    if j == DEFERRED:
                        break
                    deferred.pop(0)
                    where[k] = j
                    queue[j].append(k)
                    log.append((t, ids[k], j))
                kick(t)
        for rid in sorted(ids):
            k = pos[rid]
            if arr[k] == t:
                push()
                j = macro.route(rid, S[k], arr[k], t)
                log.append((t, rid, j))
                if j == DEFERRED:
                    deferred.append(k)
                else:
                    where[k] = j
                    queue[j].append(k)
                kick(t)
        if all(d >= 0 for d in done):
            break
        if all(e < 0 for e in end) and all(a <= t for a in arr):
            break                      # quiescent: only never-admissible requests remain
        t += tick
    recs = {ids[k]: dict(inst=where[k], t_first_ns=first[k], t_decode_begin_ns=dbeg[k],
                         t_done_ns=done[k], n_gen=ngen[k]) for k in range(n)}
    return recs, log, preempts
