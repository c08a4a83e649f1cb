"""TP=2 instance pair on two B200s: prefill + decode
throughput of the 70B shape (configs[3]: Llama-2-70B, TP=2) with the residual
all-reduce either fused with the residual add and RMSNorm over NVLink peer memory
(default) or as NCCL all-reduce + separate RMSNorm (ECOSERVE_TP_FUSED=0).

  python tools/tp_bench.py [--layers 80] [--batch 128] [--prompt 1024] [--steps 16]

One process per GPU (spawn); random-init weights drawn per rank directly in the
local (sharded) shapes; device time from the instance's phase events, max over ranks.
"""
import argparse
import dataclasses
import json
import os
import sys

import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(rank, nid, args, q):
    try:
        import numpy as np
        from paper_2504_18154_b200.instance import Instance, random_device_weights
        from synthetic.shapes import get_shape
        torch.cuda.set_device(rank)
        dev = torch.device("cuda", rank)
        shape = get_shape("70b").with_layers(args.layers)
        local = dataclasses.replace(shape, n_heads=shape.n_heads // 2, n_kv_heads=shape.n_kv_heads // 2,
                                    ffn_dim=shape.ffn_dim // 2, tp_size=1)
        # --tp1: one rank's shard as a plain TP=1 instance (no exchange) -- the comm-free floor
        shape = local if args.tp1 else dataclasses.replace(shape, tp_size=2)
        tp_kw = {} if args.tp1 else dict(tp_size=2, tp_rank=rank, nccl_id=nid)
        w = random_device_weights(local, seed=7 + rank, device=dev)
        # replicated tensors must match across the pair
        g = torch.Generator(device=dev)
        g.manual_seed(1234)
        for k in ("embed", "lm_head"):
            w[k] = (torch.randn(w[k].shape, generator=g, device=dev) * 0.02).to(torch.bfloat16)
        w["final_norm"] = torch.ones_like(w["final_norm"])
        for lw in w["layers"]:
            for k in ("attn_norm", "ffn_norm"):
                lw[k] = torch.ones_like(lw[k])
        blocks = args.batch * ((args.prompt + args.steps * (args.reps + 1) + 63) // 64 + 1) + 64
        inst = Instance(shape, w, blocks, rank, token_budget=16384, max_batch=max(256, args.batch),
                        max_positions=args.prompt + 1024, free_raw_after_create=True, **tp_kw)
        rng = np.random.default_rng(0)
        ids = list(range(args.batch))
        out = {}
        for rep in range(args.reps + 1):  # rep 0 = warmup
            base = 100000 * (rep + 1)
            inst.timing(reset=True)
            for i in range(0, args.batch, 16):
                inst.prefill([(base + j, rng.integers(0, shape.vocab, args.prompt).astype(np.int32), 512)
                              for j in ids[i:i + 16]])
            inst.decode([base + j for j in ids], args.steps)
            t = inst.timing(reset=True)
            inst.release([base + j for j in ids])
            if rep > 0:
                for k in ("prefill_ms", "decode_ms"):
                    out[k] = min(out.get(k, 1e30), t[k])
        if args.ncu:  # one decode step inside a profiler range (ncu --profile-from-start off)
            base = 100000 * (args.reps + 3)
            for i in range(0, args.batch, 16):
                inst.prefill([(base + j, rng.integers(0, shape.vocab, args.prompt).astype(np.int32), 512)
                              for j in ids[i:i + 16]])
            inst.decode([base + j for j in ids], 1)
            torch.cuda.synchronize()
            torch.cuda.cudart().cudaProfilerStart()
            inst.decode([base + j for j in ids], 1)
            torch.cuda.synchronize()
            torch.cuda.cudart().cudaProfilerStop()
            inst.release([base + j for j in ids])
        if args.profile:  # one more rep with per-kernel-class events (breaks PDL overlap: shares only)
            inst.set_profiling(2)
            base = 100000 * (args.reps + 2)
            inst.timing(reset=True)
            for i in range(0, args.batch, 16):
                inst.prefill([(base + j, rng.integers(0, shape.vocab, args.prompt).astype(np.int32), 512)
                              for j in ids[i:i + 16]])
            inst.decode([base + j for j in ids], args.steps)
            out["classes"] = {k: round(v, 3) if isinstance(v, float) else v
                              for k, v in inst.timing(reset=True).items()}
            inst.release([base + j for j in ids])
        inst.close()
        q.put((rank, out, None))
    except Exception as e:  # surface to the parent
        import traceback
        q.put((rank, None, traceback.format_exc()))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=80)
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--prompt", type=int, default=1024)
    ap.add_argument("--steps", type=int, default=16)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--profile", action="store_true", help="add a per-kernel-class pass (rank 0's classes)")
    ap.add_argument("--ncu", action="store_true", help="profiler range around one decode step")
    ap.add_argument("--tp1", action="store_true", help="one rank's shard as a TP=1 instance on one GPU")
    args = ap.parse_args()
    from paper_2504_18154_b200 import build as B
    B.build(verbose=False)
    from paper_2504_18154_b200.instance import nccl_unique_id
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    nid = nccl_unique_id()
    nproc = 1 if args.tp1 else 2
    ps = [ctx.Process(target=worker, args=(r, nid, args, q)) for r in range(nproc)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(nproc):
        r, out, err = q.get(timeout=1800)
        if err:
            print(err, file=sys.stderr)
            sys.exit(1)
        res[r] = out
    for p in ps:
        p.join()
    pre = max(res[r]["prefill_ms"] for r in res)
    dec = max(res[r]["decode_ms"] for r in res)
    line = {"config": {"shape": f"70b-L{args.layers} " + ("rank shard as TP=1" if args.tp1 else "TP=2"), "batch": args.batch, "prompt": args.prompt,
                       "decode_steps": args.steps},
            "allreduce": "nccl+rmsnorm" if os.environ.get("ECOSERVE_TP_FUSED") == "0" else "fused-p2p",
            "prefill_ms": round(pre, 3), "decode_ms": round(dec, 3),
            "prefill_tok_s": round(args.batch * args.prompt / (pre * 1e-3), 1),
            "decode_tok_s": round(args.batch * args.steps / (dec * 1e-3), 1),
            "decode_ms_per_step": round(dec / args.steps, 3)}
    if args.profile:
        line["classes_rank0"] = res[0]["classes"]
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
