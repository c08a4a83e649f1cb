"""In-step cost of each kernel class of the 8B decode step (B = 128, contexts of the
bench's running set), measured by difference: the same decode phase with kernels
dropped through ECOSERVE_ABLATE (timing only; tokens are meaningless then).
  python tools/decode_ablate.py            # runs every variant in a subprocess
  python tools/decode_ablate.py --one      # one run with the current environment
Prints one JSON line per variant: device ms per decode step (phase events) and wall."""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def one(B=128, steps=16, reps=3, shape_name="8b"):
    import torch
    from paper_2504_18154_b200.instance import Instance, random_device_weights
    from synthetic.shapes import get_shape
    from synthetic.traces import make_trace
    shape = get_shape(shape_name)
    dev = torch.device("cuda", 0)
    w = random_device_weights(shape, seed=1000, device=dev)
    inst = Instance(shape, w, 6000, 0, token_budget=16384, max_batch=256, max_positions=8192,
                    free_raw_after_create=True)
    torch.cuda.empty_cache()
    trace = make_trace("8b-cycle", B, seed=1, vocab=shape.vocab)
    for i in range(0, B, 32):
        inst.prefill([(r.req_id, r.prompt, 4096) for r in trace[i:i + 32]])
    ids = [r.req_id for r in trace]
    inst.decode(ids, 2)
    res = []
    for _ in range(reps):
        inst.set_profiling(1)
        inst.timing(reset=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        inst.decode(ids, steps)
        wall = time.perf_counter() - t0
        tm = inst.timing(reset=True)
        res.append((tm["decode_ms"] / steps, 1e3 * wall / steps))
    ctx = sum(r.prompt_len for r in trace) / B
    best = min(res)
    print(json.dumps({"ablate": int(os.environ.get("ECOSERVE_ABLATE", "0")), "env": {k: v for k, v in os.environ.items()
                      if k.startswith("ECOSERVE_")}, "B": B, "mean_ctx": round(ctx, 1),
                      "dev_ms_per_step": round(best[0], 4), "wall_ms_per_step": round(best[1], 4),
                      "all": [[round(a, 4), round(b, 4)] for a, b in res]}), flush=True)
    inst.close()


if __name__ == "__main__":
    if "--one" in sys.argv:
        one()
    else:
        extra = [a for a in sys.argv[1:] if "=" in a]
        variants = [{}, {"ECOSERVE_ABLATE": "1"}, {"ECOSERVE_ABLATE": "2"}, {"ECOSERVE_ABLATE": "4"},
                    {"ECOSERVE_ABLATE": "7"}]
        for e in extra:
            k, v = e.split("=", 1)
            variants.append({k: v})
        for v in variants:
            env = {**os.environ, **v}
            subprocess.run([sys.executable, os.path.abspath(__file__), "--one"], env=env, timeout=900)
