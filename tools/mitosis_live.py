"""Mitosis live on B200s (BASELINE configs[4]; Fig. 10):
a macro instance serves a long-prompt Poisson trace whose rate steps up and back down;
with --resize the macro grows when the rate steps up and contracts afterwards (the drained
instances' running requests move with their paged KV over NVLink). Reports joint
TTFT/TPOT attainment per window (every 30 s), migrations and their time, against the
same trace on a static macro of the small and of the full size.

  python tools/mitosis_live.py --gpus 4 --shape 34b --rates 2,5,2 --step-s 40 --window-s 20
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def stepped_trace(preset, rates, step_s, vocab, seed=1):
    from synthetic.traces import make_trace
    out, rid = [], 0
    for k, rate in enumerate(rates):
        n = max(1, int(rate * step_s * 1.5))
        tr = make_trace(preset, n, seed=seed + k, rate_per_s=rate, vocab=vocab)
        for r in tr:
            if r.arrival_ns >= step_s * 1e9:
                break
            r.arrival_ns += int(k * step_s * 1e9)
            r.req_id = rid
            rid += 1
            out.append(r)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=4)
    ap.add_argument("--shape", default="34b")
    ap.add_argument("--preset", default="long")
    ap.add_argument("--rates", default="2,5,2")
    ap.add_argument("--step-s", type=float, default=40.0)
    ap.add_argument("--window-s", type=float, default=20.0)
    ap.add_argument("--slo-ttft", type=float, default=15.0)
    ap.add_argument("--slo-tpot", type=float, default=0.1)
    ap.add_argument("--max-out", type=int, default=512)
    ap.add_argument("--blocks", type=int, default=5000)
    ap.add_argument("--contract-delay-s", type=float, default=20.0)
    ap.add_argument("--only", default="", help="comma list of runs (static-small, static-full, mitosis, mitosis-auto)")
    args = ap.parse_args()
    import torch
    from paper_2504_18154_b200 import build as B
    B.build(verbose=False)
    from paper_2504_18154_b200 import metrics as MX
    from paper_2504_18154_b200.instance import Instance, random_device_weights
    from paper_2504_18154_b200.serve import PaDGServer, profile_prefill
    from synthetic.shapes import get_shape
    shape = get_shape(args.shape)
    n = min(args.gpus, torch.cuda.device_count())
    insts = []
    for g in range(n):
        dev = torch.device("cuda", g)
        torch.cuda.set_device(dev)
        insts.append(Instance(shape, random_device_weights(shape, seed=100 + g, device=dev), args.blocks, g,
                              token_budget=16384, max_batch=512, max_positions=8192 + args.max_out,
                              free_raw_after_create=True))
    lens, ns = profile_prefill(insts[0], lens=(512, 2048, 4096, 8192), vocab=shape.vocab)
    rates = [float(x) for x in args.rates.split(",")]
    trace = stepped_trace(args.preset, rates, args.step_s, shape.vocab)
    for r in trace:
        r.output_len = min(r.output_len, args.max_out)
    slo_t, slo_p = int(args.slo_ttft * 1e9), int(args.slo_tpot * 1e9)
    small = max(1, n // 2)
    # grow to n when the rate steps up; contract back to n/2 once the load has been low for a
    # while after the step down ("sustained resource underutilization")
    t_c = 2 * args.step_s + args.contract_delay_s
    runs = [("static-small", [(0, small)]), ("static-full", None),
            ("mitosis", [(0, small), (args.step_s, n), (t_c, small)]),
            # the paper's triggers: expand while requests stay Deferred, contract after
            # a quiet period (serve.PaDGServer._auto_resize)
            ("mitosis-auto", dict(n_min=small, n_max=n, n_start=small, up_s=1.0, down_s=15.0, down_live=4,
                                  cooldown_s=5.0))]
    if args.only:
        runs = [x for x in runs if x[0] in args.only.split(",")]
    for name, resize in runs:
        srv = PaDGServer(insts, slo_t, slo_p, reserve_tokens=64, predictor_table=(lens, ns), resize=resize)
        out = srv.run(trace, timeout_s=len(rates) * args.step_s + 600)
        t0 = min(r.arrival_ns for r in out.values())
        wins = {}
        for r in out.values():
            ok = MX.request_ok(r.arrival_ns, r.t_first_ns, r.t_decode_begin_ns, r.t_done_ns, r.G, slo_t, slo_p)
            wins.setdefault(int((r.arrival_ns - t0) / (args.window_s * 1e9)), []).append(ok)
        line = {"run": name, "shape": args.shape, "gpus": n, "rates": rates, "step_s": args.step_s,
                "slo": [args.slo_ttft, args.slo_tpot], "n_req": len(out),
                "attainment": round(MX.attainment([MX.request_ok(r.arrival_ns, r.t_first_ns, r.t_decode_begin_ns,
                                                                 r.t_done_ns, r.G, slo_t, slo_p)
                                                   for r in out.values()]), 4),
                "window_attainment": [round(MX.attainment(wins[k]), 3) for k in sorted(wins)],
                "migrated": sum(w.n_migrated_out for w in srv.workers),
                "migrate_ms": round(sum(w.migrate_ns for w in srv.workers) / 1e6, 2),
                "resize_log_s": [(round((t - srv.resize_log[0][0]) / 1e9, 2), a, b) for t, a, b in srv.resize_log],
                "per_instance": [sum(1 for r in out.values() if r.inst == i) for i in range(n)]}
        print(json.dumps(line), flush=True)
    for i in insts:
        i.close()


if __name__ == "__main__":
    main()
