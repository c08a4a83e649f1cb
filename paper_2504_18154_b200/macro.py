"""Python binding of the host macro-instance scheduler (include/ecoserve.h,
Alg. 1/2 of PAPER.md P:476-540) and its virtual-clock DES mode."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _lib as L

# Fixed integer cost model defaults (8B at 60% bf16 / 70% HBM of B200)
COST_DEFAULT = dict(a=2_000_000, b=14_320_000, c=270, d=3_280_000, e=1_000, f=28_600)


@dataclass
class SchedConfig:
    n_instances: int
    slo_ttft_ns: int
    slo_tpot_ns: int
    reserve_tokens: int
    total_blocks: Sequence[int]
    probe_printed: bool = False
    cost_a_ns: int = COST_DEFAULT["a"]
    cost_b_ps: int = COST_DEFAULT["b"]
    cost_c_ps: int = COST_DEFAULT["c"]
    table: Optional[Tuple[Sequence[int], Sequence[int]]] = None   # (lens, ns) piecewise-linear predictor

    def to_c(self):
        keep = []
        tb = np.ascontiguousarray(self.total_blocks, dtype=np.int64)
        keep.append(tb)
        n_table = 0
        tl = tn = None
        if self.table is not None:
            tl = np.ascontiguousarray(self.table[0], dtype=np.int64)
            tn = np.ascontiguousarray(self.table[1], dtype=np.int64)
            keep += [tl, tn]
            n_table = len(tl)
        cfg = L.MacroConfig(self.n_instances, self.slo_ttft_ns, self.slo_tpot_ns, self.reserve_tokens, 64,
                            1 if self.probe_printed else 0, self.cost_a_ns, self.cost_b_ps, self.cost_c_ps, n_table,
                            tl.ctypes.data_as(L.PI64) if tl is not None else None,
                            tn.ctypes.data_as(L.PI64) if tn is not None else None, tb.ctypes.data_as(L.PI64))
        return cfg, keep


class MacroScheduler:
    def __init__(self, cfg: SchedConfig):
        self.lib = L.load()
        self.cfg = cfg
        c, self._keep = cfg.to_c()
        h = C.c_void_p()
        L.check(self.lib.ecoserve_macro_create(C.byref(c), C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.ecoserve_macro_destroy(self.h)
            self.h = None

    def route(self, req_id: int, arrival_ns: int, prompt_len: int, now_ns: int):
        """-> (instance or -1, [Alg. 2 outcome per probed instance])"""
        inst = C.c_int32()
        outc = (C.c_int32 * self.cfg.n_instances)()
        n = C.c_int32()
        L.check(self.lib.ecoserve_macro_route(self.h, C.byref(L.RouteReq(req_id, arrival_ns, prompt_len)), now_ns,
                                              C.byref(inst), outc, C.byref(n)))
        return inst.value, list(outc[:n.value])

    def check(self, inst: int, prompt_len: int, arrival_ns: int, now_ns: int) -> int:
        r = C.c_int32()
        L.check(self.lib.ecoserve_macro_check(self.h, inst, C.byref(L.RouteReq(0, arrival_ns, prompt_len)), now_ns,
                                              C.byref(r)))
        return r.value

    def defer(self, req_id: int, arrival_ns: int, prompt_len: int) -> None:
        L.check(self.lib.ecoserve_macro_defer(self.h, C.byref(L.RouteReq(req_id, arrival_ns, prompt_len))))

    def update_status(self, inst: int, phase: int, t_switch_ns: int, total_blocks: int, reqs, alive: bool = True):
        """reqs: iterable of (req_id, arrival_ns, prompt_len, t_first_ns, n_generated, finished)."""
        reqs = list(reqs)
        arr = (L.SchedReq * max(1, len(reqs)))()
        for i, r in enumerate(reqs):
            arr[i] = L.SchedReq(int(r[0]), int(r[1]), int(r[2]), int(r[3]), int(r[4]), 1 if r[5] else 0)
        st = L.SchedStatus(phase, t_switch_ns, total_blocks, 1 if alive else 0)
        L.check(self.lib.ecoserve_macro_update_status(self.h, inst, C.byref(st), arr, len(reqs)))

    def drain_deferred(self, now_ns: int, cap: int = 4096) -> List[Tuple[int, int]]:
        out = (L.Routed * cap)()
        n = C.c_int32()
        L.check(self.lib.ecoserve_macro_drain_deferred(self.h, now_ns, out, cap, C.byref(n)))
        return [(out[i].req_id, out[i].instance) for i in range(n.value)]

    @property
    def prev_idx(self) -> int:
        return self.lib.ecoserve_macro_prev_idx(self.h)

    def predict_prefill_ns(self, S: int) -> int:
        return self.lib.ecoserve_macro_predict_prefill_ns(self.h, S)


def mitosis_step(sizes: Sequence[int], n_l: int, n_u: int, expand: bool):
    """One mitosis expansion / contraction step (C++). Returns (new sizes, (kind, a1, a2))."""
    lib = L.load()
    cap = len(sizes) + 1
    arr = (C.c_int32 * cap)(*sizes)
    n = C.c_int32(len(sizes))
    act = (C.c_int32 * 3)()
    L.check(lib.ecoserve_mitosis_step(arr, C.byref(n), cap, n_l, n_u, 1 if expand else 0, act))
    return list(arr[:n.value]), tuple(act)


def handler_to_bytes(actor_id: int, device: int, tp_size: int, tp_rank: int, kv_blocks: int, address: str) -> bytes:
    lib = L.load()
    h = L.InstanceHandler(actor_id, device, tp_size, tp_rank, kv_blocks, address.encode())
    need = -lib.ecoserve_handler_serialize(C.byref(h), None, 0)
    buf = (C.c_uint8 * need)()
    n = lib.ecoserve_handler_serialize(C.byref(h), buf, need)
    if n != need:
        raise L.EcoError(L.ERR_INVALID_ARG, "serialize")
    return bytes(buf)


def handler_from_bytes(b: bytes) -> dict:
    lib = L.load()
    buf = (C.c_uint8 * len(b)).from_buffer_copy(b)
    h = L.InstanceHandler()
    L.check(lib.ecoserve_handler_deserialize(buf, len(b), C.byref(h)))
    return dict(actor_id=h.actor_id, device=h.device, tp_size=h.tp_size, tp_rank=h.tp_rank, kv_blocks=h.kv_blocks,
                address=h.address.decode())


def des_run(cfg: SchedConfig, arrival_ns, prompt_len, output_len, cost_d_ns=COST_DEFAULT["d"],
            cost_e_ns=COST_DEFAULT["e"], cost_f_ps=COST_DEFAULT["f"], token_budget: int = 16384):
    """Virtual-clock DES of the macro instance (C++). Returns dict of per-request
    arrays (inst, t_first, t_decode_begin, t_done, n_preempt) and the route log [(t, req, inst)]."""
    lib = L.load()
    c, keep = cfg.to_c()
    n = len(arrival_ns)
    a = np.ascontiguousarray(arrival_ns, dtype=np.int64)
    s = np.ascontiguousarray(prompt_len, dtype=np.int32)
    g = np.ascontiguousarray(output_len, dtype=np.int32)
    inst = np.zeros(n, np.int32)
    npre = np.zeros(n, np.int32)
    tf, tb, td = np.zeros(n, np.int64), np.zeros(n, np.int64), np.zeros(n, np.int64)
    cap = 8 * n + 16
    log = np.zeros((cap, 3), np.int64)
    nlog = C.c_int32()
    d = L.DesConfig(cost_d_ns, cost_e_ns, cost_f_ps, token_budget)
    L.check(lib.ecoserve_des_run(C.byref(c), C.byref(d), a.ctypes.data_as(L.PI64), s.ctypes.data_as(L.PI32),
                                 g.ctypes.data_as(L.PI32), n, inst.ctypes.data_as(L.PI32), tf.ctypes.data_as(L.PI64),
                                 tb.ctypes.data_as(L.PI64), td.ctypes.data_as(L.PI64), log.ctypes.data_as(L.PI64),
                                 cap, C.byref(nlog), npre.ctypes.data_as(L.PI32)))
    return dict(inst=inst, t_first=tf, t_decode_begin=tb, t_done=td, n_preempt=npre,
                route_log=[tuple(int(v) for v in row) for row in log[:min(cap, nlog.value)]])
