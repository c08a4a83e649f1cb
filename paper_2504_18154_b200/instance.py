"""Python-side handle of one PaDG instance (include/ecoserve.h).

PyTorch is used only as the device-memory allocator for the buffers the C ABI
borrows (weights, prepared weights, KV pool); every computation runs in
libecoserve.so.
"""
from __future__ import annotations

import ctypes as C
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np
import torch

from . import _lib as L

LAYER_TENSORS = ("attn_norm", "wq", "wk", "wv", "wo", "ffn_norm", "w_gate", "w_up", "w_down")


def c_shape(s, tp_size: int = 1) -> L.ModelShape:
    return L.ModelShape(s.n_layers, s.hidden, s.n_heads, s.n_kv_heads, s.head_dim, s.ffn_dim, s.vocab,
                        float(s.rope_theta), float(s.rms_eps), tp_size)


def upload_bf16(bits: np.ndarray, device) -> torch.Tensor:
    """uint16 bf16 bit patterns (host) -> torch.bfloat16 tensor on `device`."""
    t = torch.from_numpy(np.ascontiguousarray(bits).view(np.int16))
    return t.to(device).view(torch.bfloat16)


def device_weights_from_host(w, device) -> Dict:
    """synthetic.weights.Bf16Weights -> dict of device bf16 tensors."""
    return {
        "embed": upload_bf16(w.embed, device),
        "lm_head": upload_bf16(w.lm_head, device),
        "final_norm": upload_bf16(w.final_norm, device),
        "layers": [{k: upload_bf16(l[k], device) for k in LAYER_TENSORS} for l in w.layers],
    }


def random_device_weights(shape, seed: int, device) -> Dict:
    """Random-init weights drawn directly on the GPU (bench only; same recipe
    as synthetic.weights but torch's CUDA generator, so not oracle-reproducible)."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    H, D, F, V = shape.hidden, shape.head_dim, shape.ffn_dim, shape.vocab
    M, Mkv = shape.n_heads, shape.n_kv_heads

    def mat(o, i, std=None):
        return (torch.randn(o, i, generator=g, device=device) * (std if std else i ** -0.5)).to(torch.bfloat16)

    def norm(n):
        return (1.0 + (torch.rand(n, generator=g, device=device) - 0.5) * 0.2).to(torch.bfloat16)
    layers = []
    for _ in range(shape.n_layers):
        layers.append({"attn_norm": norm(H), "wq": mat(M * D, H), "wk": mat(Mkv * D, H), "wv": mat(Mkv * D, H),
                       "wo": mat(H, M * D), "ffn_norm": norm(H), "w_gate": mat(F, H), "w_up": mat(F, H),
                       "w_down": mat(H, F)})
    return {"embed": mat(V, H, 1.0), "lm_head": mat(V, H, 2.0 / H ** 0.5), "final_norm": norm(H), "layers": layers}


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    L.check(L.load().ecoserve_nccl_unique_id(buf))
    return buf.raw


def shard_weights(w: Dict, shape, tp: int, rank: int) -> Dict:
    """TP shard of full weights: heads [r*M/tp, (r+1)*M/tp), kv heads
    [r*Mkv/tp, ..), FFN columns [r*F/tp, ..); embed / LM head / norms replicated."""
    D = shape.head_dim
    mq, mk, f = shape.n_heads // tp * D, shape.n_kv_heads // tp * D, shape.ffn_dim // tp
    out = {k: w[k] for k in ("embed", "lm_head", "final_norm")}
    out["layers"] = []
    for l in w["layers"]:
        out["layers"].append({
            "attn_norm": l["attn_norm"], "ffn_norm": l["ffn_norm"],
            "wq": l["wq"][rank * mq:(rank + 1) * mq].contiguous(),
            "wk": l["wk"][rank * mk:(rank + 1) * mk].contiguous(),
            "wv": l["wv"][rank * mk:(rank + 1) * mk].contiguous(),
            "wo": l["wo"][:, rank * mq:(rank + 1) * mq].contiguous(),
            "w_gate": l["w_gate"][rank * f:(rank + 1) * f].contiguous(),
            "w_up": l["w_up"][rank * f:(rank + 1) * f].contiguous(),
            "w_down": l["w_down"][:, rank * f:(rank + 1) * f].contiguous()})
    return out


class Instance:
    """One instance on one GPU. Owns (via torch) the borrowed buffers."""

    def __init__(self, shape, weights: Dict, num_blocks: int, device: int = 0, token_budget: int = 16384,
                 max_batch: int = 512, max_positions: int = 16384, debug_hidden: bool = False,
                 free_raw_after_create: bool = False, stream: Optional[int] = None, tp_size: int = 1,
                 tp_rank: int = 0, nccl_id: Optional[bytes] = None):
        """tp_size 2: `weights` hold this rank's shard (see shard_weights); all
        ranks of the pair construct concurrently with the same nccl_id."""
        self.lib = L.load()
        self.shape = shape
        self.device = torch.device("cuda", device)
        self.cshape = c_shape(shape, tp_size)
        self._nccl_id = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        pool_bytes = self.lib.ecoserve_kv_pool_bytes(C.byref(self.cshape), 64, num_blocks)
        prep_bytes = self.lib.ecoserve_prepared_weight_bytes(C.byref(self.cshape))
        if pool_bytes < 0 or prep_bytes < 0:
            raise L.EcoError(L.ERR_INVALID_ARG, "unsupported shape")
        self.pool = torch.empty(pool_bytes, dtype=torch.uint8, device=self.device)
        self.prepared = torch.empty(prep_bytes, dtype=torch.uint8, device=self.device)
        self.weights = weights
        ptrs = []
        for l in weights["layers"]:
            ptrs += [l[k].data_ptr() for k in LAYER_TENSORS]
        self._layer_ptrs = (C.c_void_p * len(ptrs))(*ptrs)
        self.cw = L.Weights(weights["embed"].data_ptr(), weights["lm_head"].data_ptr(),
                            weights["final_norm"].data_ptr(), C.cast(self._layer_ptrs, C.POINTER(C.c_void_p)))
        self.ckv = L.KVPool(64, num_blocks, self.pool.data_ptr())
        self.cfg = L.EngineConfig(token_budget, max_batch, max_positions, 1 if debug_hidden else 0)
        self.num_blocks = num_blocks
        h = C.c_void_p()
        torch.cuda.set_device(self.device)
        L.check(self.lib.ecoserve_instance_create(C.byref(self.cshape), C.byref(self.ckv), C.byref(self.cw),
                                                  C.c_void_p(self.prepared.data_ptr()), device, tp_rank,
                                                  self._nccl_id, C.c_void_p(stream) if stream else None,
                                                  C.byref(self.cfg), C.byref(h)))
        self.h = h
        if free_raw_after_create:  # wq/wk/wv/w_gate/w_up were copied into the prepared buffer
            for l in weights["layers"]:
                for k in ("wq", "wk", "wv", "w_gate", "w_up"):
                    l[k] = None

    def close(self):
        if getattr(self, "h", None):
            self.lib.ecoserve_instance_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ phases
    def prefill(self, reqs: Sequence[Tuple[int, np.ndarray, int]]) -> np.ndarray:
        """reqs: (req_id, prompt int32[S], max_new_tokens). Returns first tokens."""
        n = len(reqs)
        arr = (L.Request * n)()
        keep = []
        for i, (rid, prompt, g) in enumerate(reqs):
            p = np.ascontiguousarray(prompt, dtype=np.int32)
            keep.append(p)
            arr[i] = L.Request(int(rid), p.ctypes.data_as(L.PI32), len(p), int(g))
        out = np.zeros(n, dtype=np.int32)
        L.check(self.lib.ecoserve_prefill_phase(self.h, arr, n, out.ctypes.data_as(L.PI32)), self.h)
        return out

    def decode(self, req_ids: Sequence[int], steps: int):
        n = len(req_ids)
        ids = np.ascontiguousarray(req_ids, dtype=np.int64)
        toks = np.zeros((n, steps), dtype=np.int32)
        nf = C.c_int32(0)
        L.check(self.lib.ecoserve_decode_phase(self.h, ids.ctypes.data_as(L.PI64), n, steps,
                                               toks.ctypes.data_as(L.PI32), C.byref(nf)), self.h)
        return toks, nf.value

    def hybrid_step(self, chunks: Sequence[Tuple[int, np.ndarray, int, int]], decode_ids: Sequence[int]):
        """One hybrid (chunked-prefill + decode) forward pass (N3, Sarathi-style).
        chunks: (req_id, full prompt int32[S], max_new_tokens, chunk_len) -- each
        continues its request's prompt; decode_ids advance one token each.
        Returns (chunk_tokens [-1 unless the chunk completed the prompt], decode_tokens)."""
        nc, nd = len(chunks), len(decode_ids)
        arr = (L.Chunk * max(nc, 1))()
        keep = []
        for i, (rid, prompt, g, clen) in enumerate(chunks):
            p = np.ascontiguousarray(prompt, dtype=np.int32)
            keep.append(p)
            arr[i] = L.Chunk(int(rid), p.ctypes.data_as(L.PI32), len(p), int(g), int(clen))
        ids = np.ascontiguousarray(decode_ids, dtype=np.int64)
        ct = np.zeros(max(nc, 1), dtype=np.int32)
        dt = np.zeros(max(nd, 1), dtype=np.int32)
        L.check(self.lib.ecoserve_hybrid_step(self.h, arr, nc, ids.ctypes.data_as(L.PI64), nd,
                                              ct.ctypes.data_as(L.PI32), dt.ctypes.data_as(L.PI32)), self.h)
        return ct[:nc], dt[:nd]

    @property
    def block_bytes(self) -> int:
        return self.lib.ecoserve_kv_pool_bytes(C.byref(self.cshape), 64, 1)

    def export_kv(self, req_id: int, device) -> tuple:
        """First half of a KV move: copy request `req_id`'s blocks into a staging
        buffer on `device` (peer copy over NVLink) and release it here. Returns the
        handle that `import_kv` of the destination instance takes (FuDG hand-off,
        SURVEY 8(f) N4(i); the destination may import from its own thread)."""
        st = L.ReqState()
        _, reqs = self.status()
        info = next(r for r in reqs if r["req_id"] == req_id)
        stage = torch.empty(max(1, info["n_blocks"]) * self.block_bytes, dtype=torch.uint8, device=device)
        prompt = np.zeros(info["prompt_len"], dtype=np.int32)
        L.check(self.lib.ecoserve_kv_export(self.h, int(req_id), C.c_void_p(stage.data_ptr()), stage.numel(),
                                            prompt.ctypes.data_as(L.PI32), len(prompt), C.byref(st)), self.h)
        self.release([req_id])
        return st, prompt, stage

    def import_kv(self, handle: tuple) -> None:
        """Second half of a KV move (see export_kv): place the staged blocks in this pool."""
        st, prompt, stage = handle
        L.check(self.lib.ecoserve_kv_import(self.h, C.byref(st), prompt.ctypes.data_as(L.PI32),
                                            C.c_void_p(stage.data_ptr())), self.h)

    def migrate_to(self, other: "Instance", req_id: int) -> dict:
        """Move a running request with its paged KV to `other` (any GPU): export
        into a staging buffer on the destination device (peer copy over NVLink),
        import there, release here (mitosis contraction / rebalancing, N1)."""
        st = L.ReqState()
        _, reqs = self.status()
        info = next(r for r in reqs if r["req_id"] == req_id)
        stage = torch.empty(max(1, info["n_blocks"]) * self.block_bytes, dtype=torch.uint8, device=other.device)
        prompt = np.zeros(info["prompt_len"], dtype=np.int32)
        L.check(self.lib.ecoserve_kv_export(self.h, int(req_id), C.c_void_p(stage.data_ptr()), stage.numel(),
                                            prompt.ctypes.data_as(L.PI32), len(prompt), C.byref(st)), self.h)
        L.check(other.lib.ecoserve_kv_import(other.h, C.byref(st), prompt.ctypes.data_as(L.PI32),
                                             C.c_void_p(stage.data_ptr())), other.h)
        self.release([req_id])
        return dict(req_id=st.req_id, n_blocks=st.n_blocks, bytes=st.n_blocks * self.block_bytes,
                    n_generated=st.n_generated)

    def release(self, req_ids: Sequence[int]) -> None:
        ids = np.ascontiguousarray(req_ids, dtype=np.int64)
        L.check(self.lib.ecoserve_release(self.h, ids.ctypes.data_as(L.PI64), len(ids)), self.h)

    def status(self, cap: int = 4096):
        st = L.InstanceStatus()
        rs = (L.ReqStatus * cap)()
        L.check(self.lib.ecoserve_get_status(self.h, C.byref(st), rs, cap), self.h)
        reqs = [dict(req_id=r.req_id, prompt_len=r.prompt_len, n_generated=r.n_generated,
                     finished=bool(r.finished), n_blocks=r.n_blocks) for r in rs[:min(cap, st.n_requests)]]
        return dict(alive=bool(st.alive), n_requests=st.n_requests, blocks_total=st.blocks_total,
                    blocks_used=st.blocks_used), reqs

    def set_profiling(self, level: int) -> None:
        L.check(self.lib.ecoserve_set_profiling(self.h, level), self.h)

    def timing(self, reset: bool = False) -> Dict:
        t = L.Timing()
        L.check(self.lib.ecoserve_get_timing(self.h, C.byref(t), 1 if reset else 0), self.h)
        return t.as_dict()

    def force_token(self, req_id: int, token: int) -> None:
        """Teacher forcing (debug instances): the next decode step of req_id feeds `token`."""
        L.check(self.lib.ecoserve_debug_force_token(self.h, int(req_id), int(token)), self.h)

    def hidden(self, req_id: int, layer: int, rows: int) -> np.ndarray:
        out = np.zeros((rows, self.shape.hidden), dtype=np.float32)
        L.check(self.lib.ecoserve_debug_hidden(self.h, int(req_id), layer, out.ctypes.data_as(L.PF32)), self.h)
        return out


class TpPairInstance:
    """One TP=2 instance of a macro instance (configs[3]: Llama-2-70B, TP=2 per
    instance): rank 0 on GPU `devices[0]`, rank 1 on
    `devices[1]`, both in this process. Every phase call runs on the two ranks
    concurrently (one thread each; the ctypes calls release the GIL) and the ranks
    meet in their fused all-reduce on the device, so the pair is driven like one
    instance by a serving worker. The ranks compute bitwise-identical tokens
    (tests/test_gpu_tp.py); rank 0's are returned. weights[r]: rank r's shard
    (shard_weights); the replicated tensors must be identical on both ranks."""

    def __init__(self, shape, weights: Sequence[Dict], num_blocks: int, devices: Sequence[int] = (0, 1), **kw):
        from concurrent.futures import ThreadPoolExecutor
        if len(devices) != 2 or len(weights) != 2:
            raise ValueError("a TP pair needs two devices and two weight shards")
        self._ex = ThreadPoolExecutor(2)
        nid = nccl_unique_id()
        futs = [self._ex.submit(Instance, shape, weights[r], num_blocks, devices[r], tp_size=2, tp_rank=r,
                                nccl_id=nid, **kw) for r in range(2)]
        self.ranks = [f.result() for f in futs]
        self.shape = shape
        self.device = self.ranks[0].device
        self.num_blocks = num_blocks

    def _both(self, name: str, *args):
        futs = [self._ex.submit(getattr(inst, name), *args) for inst in self.ranks]
        res = [f.result() for f in futs]  # re-raises a rank's EcoError
        return res[0]

    def prefill(self, reqs):
        return self._both("prefill", reqs)

    def decode(self, req_ids, steps: int):
        return self._both("decode", req_ids, steps)

    def release(self, req_ids) -> None:
        self._both("release", req_ids)

    def status(self, cap: int = 4096):
        return self.ranks[0].status(cap)

    def set_profiling(self, level: int) -> None:
        self._both("set_profiling", level)

    def timing(self, reset: bool = False) -> Dict:
        return self._both("timing", reset)

    def close(self):
        for inst in getattr(self, "ranks", []):
            inst.close()
        if getattr(self, "_ex", None):
            self._ex.shutdown(wait=True)
            self._ex = None
