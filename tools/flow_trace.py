"""Summarise ECOSERVE_FLOW_TRACE output (per-CTA %globaltimer marks of one decode-flow
launch per step, decode_flow.cu fl_mark): median / max over CTAs of each mark, us.
  python tools/flow_trace.py trace.txt"""
import collections
import sys

import numpy as np

NAMES = ["start", "first weights", "O mma done", "GU mma done", "down mma done", "epi O done", "epi GU done",
         "epi down done", "first GU act load", "first down act load", "end", "O last-arriver go",
         "O reducer chunk0 loads", "O reducer chunk0 stores", "O reducer all chunks", "O reducer chunk0 slots"]


GU_NAMES = ["start", "first stage", "last MMA", "tail published", "head flag seen", "head partial landed",
            "epilogue done", "end"]


def main(path):
    names = GU_NAMES if "--gu" in sys.argv else NAMES
    runs, cur = [], None
    for line in open(path):
        if line.startswith("#"):
            cur = collections.defaultdict(list)
            runs.append(cur)
            continue
        c, k, t = line.split()
        cur[int(k)].append(int(t) / 1e3)
    r = runs[-1]
    print(f"{len(runs)} traced launches; the last one:")
    for k, n in enumerate(names):
        v = np.array(r.get(k, []))
        if len(v):
            print(f"  {k:2d} {n:22s} min {v.min():8.2f}  med {np.median(v):8.2f}  max {v.max():8.2f} us  ({len(v)} CTAs)")


if __name__ == "__main__":
    main([a for a in sys.argv[1:] if not a.startswith("--")][0])
