"""Summarise ECOSERVE_GW_TRACE (per-CTA marks of the 4 decode GEMMs of the gate/up waves
path, layer 5): per kernel, min / median / max over CTAs of each mark (us)."""
import collections
import sys

import numpy as np

K = ["GU wave 1", "down K part 1", "GU wave 2", "down K part 2"]
M = ["CTA start", "prologue done", "first stage", "last MMA", "epilogue done", "acc ready", "last load", "-"]
runs, cur = [], None
for line in open(sys.argv[1]):
    if line.startswith("#"):
        cur = collections.defaultdict(list)
        runs.append(cur)
        continue
    k, c, m, t = map(int, line.split())
    cur[(k, m)].append(t / 1e3)
r = runs[-1]
for k in range(4):
    print(K[k])
    for m in range(7):
        v = np.array(r.get((k, m), []))
        if len(v):
            print(f"   {M[m]:14s} min {v.min():7.2f} med {np.median(v):7.2f} max {v.max():7.2f}  ({len(v)})")
