#!/usr/bin/env python
"""Goodput under SLO of a live PaDG macro instance on real B200 instances
(the second half of BASELINE.json's metric: "goodput req/s at TTFT/TPOT SLO, 1-8 GPU").

One process, one worker thread per GPU instance (ctypes calls release the GIL),
the C++ macro scheduler routing in real time (Alg. 1/2 with the on-box prefill
profile as predictor, reading A13). Each probe replays a fresh Poisson trace
 shaped like ShareGPT (Table 4; prompts <= 4096 as P:660, outputs
capped at --max-out), measures joint TTFT/TPOT attainment (Sec. 3.3), and the
rate is bisected for the largest one meeting the percentile.

  python goodput_bench.py --gpus N [--shape 8b] [--p 0.9] [--n-req 300]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def srv_prefill(args, n: int) -> int:
    return args.fudg_prefill if 0 < args.fudg_prefill < n else n // 2


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--instances-per-gpu", type=int, default=1)
    ap.add_argument("--shape", default="8b")
    ap.add_argument("--preset", default="sharegpt")
    ap.add_argument("--slo-ttft", type=float, default=5.0)
    ap.add_argument("--slo-tpot", type=float, default=0.1)
    ap.add_argument("--p", type=float, default=0.9)
    ap.add_argument("--n-req", type=int, default=300)
    ap.add_argument("--duration", type=float, default=0.0,
                    help="> 0: requests per probe = max(n_req, rate x duration), so a probe measures a steady "
                         "state instead of absorbing one burst")
    ap.add_argument("--max-out", type=int, default=1024)
    ap.add_argument("--lo", type=float, default=4.0)
    ap.add_argument("--hi", type=float, default=160.0)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--blocks", type=int, default=8000)
    ap.add_argument("--rates", type=str, default="", help="comma list: fixed probes instead of bisection")
    ap.add_argument("--policy", choices=("padg", "nodg", "sarathi", "fudg"), default="padg",
                    help="padg: macro routing + rolling activation; nodg: round-robin separate batching; "
                         "sarathi: round-robin hybrid (chunked-prefill) batching; fudg: prefill-only and "
                         "decode-only instances with the KV moved over NVLink")
    ap.add_argument("--fudg-prefill", type=int, default=0, help="fudg: prefill instances (default half)")
    ap.add_argument("--chunk-budget", type=int, default=1024, help="sarathi: tokens per hybrid iteration")
    ap.add_argument("--tp", type=int, choices=(1, 2), default=1,
                    help="2: every instance is a TP=2 pair of GPUs (configs[3], e.g. --shape 70b), padg only")
    args = ap.parse_args()

    import torch

    from paper_2504_18154_b200 import build as B
    B.build(verbose=False)
    from paper_2504_18154_b200 import metrics as MX
    from paper_2504_18154_b200.instance import Instance, random_device_weights
    from paper_2504_18154_b200.serve import PaDGServer, profile_prefill
    from synthetic.shapes import get_shape
    from synthetic.traces import make_trace

    shape = get_shape(args.shape)
    n_gpu = min(args.gpus, torch.cuda.device_count())
    insts = []
    if args.tp == 2:
        import dataclasses

        from paper_2504_18154_b200.instance import TpPairInstance
        assert args.policy == "padg" and n_gpu >= 2
        n_gpu -= n_gpu % 2
        local = dataclasses.replace(shape, n_heads=shape.n_heads // 2, n_kv_heads=shape.n_kv_heads // 2,
                                    ffn_dim=shape.ffn_dim // 2, tp_size=1)
        for g in range(0, n_gpu, 2):
            ws = []
            for r in range(2):
                dev = torch.device("cuda", g + r)
                torch.cuda.set_device(dev)
                w = random_device_weights(local, seed=100 + g + r, device=dev)
                gen = torch.Generator(device=dev)  # replicated tensors: identical on both ranks
                gen.manual_seed(4321 + g)
                for k in ("embed", "lm_head"):
                    w[k] = (torch.randn(w[k].shape, generator=gen, device=dev) * 0.02).to(torch.bfloat16)
                w["final_norm"] = torch.ones_like(w["final_norm"])
                ws.append(w)
            insts.append(TpPairInstance(dataclasses.replace(shape, tp_size=2), ws, args.blocks, (g, g + 1),
                                        token_budget=16384, max_batch=512, max_positions=8192 + args.max_out,
                                        free_raw_after_create=True))
    for g in range(n_gpu if args.tp == 1 else 0):
        dev = torch.device("cuda", g)
        torch.cuda.set_device(dev)
        w = random_device_weights(shape, seed=100 + g, device=dev)
        for _ in range(args.instances_per_gpu):
            insts.append(Instance(shape, w, args.blocks, g, token_budget=16384, max_batch=512,
                                  max_positions=8192 + args.max_out, free_raw_after_create=(args.instances_per_gpu == 1)))
    lens, ns = profile_prefill(insts[0], vocab=shape.vocab)
    slo_ttft, slo_tpot = int(args.slo_ttft * 1e9), int(args.slo_tpot * 1e9)
    probes = []
    rid0 = [0]

    def attain_at(rate: float) -> float:
        n_req = max(args.n_req, int(rate * args.duration))
        trace = make_trace(args.preset, n_req, seed=int(rate * 1000) % 100003, rate_per_s=rate, vocab=shape.vocab)
        for r in trace:
            r.output_len = min(r.output_len, args.max_out)
            r.req_id += rid0[0]
        rid0[0] += n_req
        for i, inst in enumerate(insts):  # the previous probe released everything it left behind
            st, _ = inst.status()
            assert st["alive"] and st["n_requests"] == 0, f"instance {i} not empty before the probe: {st}"
        srv = PaDGServer(insts, slo_ttft, slo_tpot, reserve_tokens=237, predictor_table=(lens, ns),
                         policy=args.policy, chunk_budget=args.chunk_budget, fudg_prefill=args.fudg_prefill)
        t0 = time.perf_counter()
        out = srv.run(trace, timeout_s=900)
        wall = time.perf_counter() - t0
        recs = [MX.request_ok(r.arrival_ns, r.t_first_ns, r.t_decode_begin_ns, r.t_done_ns, r.G, slo_ttft, slo_tpot)
                for r in out.values()]
        att = MX.attainment(recs)
        fin = [x for x in recs if x["finished"]]
        toks = sum(r.G for r in out.values() if r.t_done_ns >= 0)
        per_inst = [sum(1 for r in out.values() if r.inst == i) for i in range(len(insts))]
        probes.append({"rate": round(rate, 3), "n_req": n_req, "attainment": round(att, 4), "wall_s": round(wall, 2),
                       "ttft_p90_s": round(float(np.percentile([x["ttft_ns"] for x in fin], 90)) / 1e9, 4) if fin else None,
                       "tpot_p90_ms": round(float(np.percentile([x["tpot_ns"] for x in fin], 90)) / 1e6, 3) if fin else None,
                       "out_tok_s": round(toks / wall, 1), "per_instance": per_inst,
                       "deferred": sum(1 for x in srv.route_log if x[2] < 0)})
        print(json.dumps({"probe": probes[-1]}), flush=True)
        return att

    if args.rates:
        for r in [float(x) for x in args.rates.split(",")]:
            attain_at(r)
        ok = [p["rate"] for p in probes if p["attainment"] >= args.p]
        gp = max(ok) if ok else 0.0
    else:
        gp = MX.bisect_goodput(attain_at, args.p, args.lo, args.hi, args.iters)
    line = {"metric": "goodput req/s at TTFT/TPOT SLO", "value": gp, "unit": "req/s", "n_gpus": n_gpu,
            "instances": len(insts), "tp": args.tp, "p": args.p, "slo": {"ttft_s": args.slo_ttft, "tpot_s": args.slo_tpot},
            "config": {"workload": f"{args.preset} Poisson, max({args.n_req}, rate x {args.duration:g} s) req/probe, "
                                   f"outputs <= {args.max_out}",
                       "shape": args.shape,
                       "macro": f"{len(insts)} instances, " + {
                           "padg": "rolling activation (Alg. 1/2)", "nodg": "NoDG round-robin separate batching",
                           "sarathi": f"NoDG round-robin hybrid batching, {args.chunk_budget}-token iterations",
                           "fudg": f"FuDG: {srv_prefill(args, len(insts))} prefill + "
                                   f"{len(insts) - srv_prefill(args, len(insts))} decode instances, KV over NVLink"}[
                           args.policy]},
            "policy": args.policy,
            "predictor": {"lens": lens, "ns": ns}, "probes": probes}
    print(json.dumps(line), flush=True)
    for i in insts:
        i.close()


if __name__ == "__main__":
    main()
