"""ORACLE (test infrastructure only) -- mitosis scaling, SURVEY 8(f) N1.

PAPER.md Sec. 3.5.1 (Fig. 7 with N_l = 3, N_u = 6): instances are
added to / removed from macro instances one at a time.

Expansion: "New instances are incrementally added until the number
of instances exceeds the upper limit N_u, at which point a new macro instance
containing N_l instances is split off from the original macro instance. If
additional instances are still required, they are first added to the original
macro instance until it again reaches N_u, and subsequent instances are then
added to the new macro instance."  Reading: add to the first macro (creation
order) that is below N_u; if every macro is full, add to the last one, which
then holds N_u + 1 and splits off a new macro of N_l (it keeps N_u + 1 - N_l).

Contraction: "instances are firstly removed from the smallest macro
instance until [it] reaches N_l. Next, instances start to be removed from a full
macro instance. When the total number of instances across these two macro
instances reaches N_u, they will be merged into a single macro instance after
one additional instance is removed."  Reading: s = the smallest macro (last in
creation order on ties); if size(s) > N_l remove from s; else the partner p is
the other partially filled macro if any, else the last full one; if
size(s) + size(p) > N_u remove one instance from p; if it equals N_u remove one
from p and merge s into p (one macro of N_u - 1). A macro at 1 instance that
must shrink is removed entirely.

Each call performs exactly one action; macro sizes are a list in creation order.
"""
from __future__ import annotations

from typing import List, Tuple


def expand(sizes: List[int], n_l: int, n_u: int) -> Tuple[List[int], tuple]:
    s = list(sizes)
    if not s:
        return [1], ("create", 0)
    for i, v in enumerate(s):
        if v < n_u:
            s[i] += 1
            return s, ("add", i)
    i = len(s) - 1
    s[i] = n_u + 1 - n_l
    s.append(n_l)
    return s, ("add_split", i, len(s) - 1)


def contract(sizes: List[int], n_l: int, n_u: int) -> Tuple[List[int], tuple]:
    s = list(sizes)
    if not s:
        raise ValueError("no instance to remove")
    if len(s) == 1:
        if s[0] == 1:
            return [], ("remove_macro", 0)
        s[0] -= 1
        return s, ("remove", 0)
    small = min(range(len(s)), key=lambda i: (s[i], -i))
    if s[small] > n_l:
        s[small] -= 1
        return s, ("remove", small)
    partial = [i for i in range(len(s)) if i != small and s[i] < n_u]
    full = [i for i in range(len(s)) if i != small and s[i] >= n_u]
    p = partial[-1] if partial else full[-1]
    total = s[small] + s[p]
    if total > n_u:
        s[p] -= 1
        return s, ("remove", p)
    # total == N_u (or below, after external changes): one more removal, then merge
    keep, gone = min(small, p), max(small, p)
    s[keep] = total - 1
    del s[gone]
    return s, ("remove_merge", p, small)
