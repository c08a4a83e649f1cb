"""ctypes binding of libecoserve.so (include/ecoserve.h, include/ecoserve_ops.h).

Argument marshalling only: every step of the hot path runs inside the CUDA
library. Loading fails loudly if the library is missing -- there is no CPU
fallback.
"""
from __future__ import annotations

import ctypes as C
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libecoserve.so")

OK, ERR_INVALID_ARG, ERR_KV_EXHAUSTED, ERR_STATE, ERR_UNSUPPORTED, ERR_CUDA, ERR_NCCL, ERR_NUMERIC = range(8)
STATUS_NAMES = {0: "OK", 1: "INVALID_ARG", 2: "KV_EXHAUSTED", 3: "STATE", 4: "UNSUPPORTED", 5: "CUDA", 6: "NCCL",
                7: "NUMERIC"}


class EcoError(RuntimeError):
    def __init__(self, status: int, msg: str = ""):
        super().__init__(f"ecoserve status {STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class ModelShape(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("hidden", C.c_int32), ("n_heads", C.c_int32),
                ("n_kv_heads", C.c_int32), ("head_dim", C.c_int32), ("ffn_dim", C.c_int32),
                ("vocab", C.c_int32), ("rope_theta", C.c_float), ("rms_eps", C.c_float), ("tp_size", C.c_int32)]


class KVPool(C.Structure):
    _fields_ = [("block_tokens", C.c_int32), ("num_blocks", C.c_int64), ("pool", C.c_void_p)]


class Weights(C.Structure):
    _fields_ = [("embed", C.c_void_p), ("lm_head", C.c_void_p), ("final_norm", C.c_void_p),
                ("layers", C.POINTER(C.c_void_p))]


class EngineConfig(C.Structure):
    _fields_ = [("token_budget", C.c_int32), ("max_batch", C.c_int32), ("max_positions", C.c_int32),
                ("debug_hidden", C.c_int32)]


class Request(C.Structure):
    _fields_ = [("req_id", C.c_int64), ("prompt", C.POINTER(C.c_int32)), ("prompt_len", C.c_int32),
                ("max_new_tokens", C.c_int32)]


class Chunk(C.Structure):
    _fields_ = [("req_id", C.c_int64), ("prompt", C.POINTER(C.c_int32)), ("prompt_len", C.c_int32),
                ("max_new_tokens", C.c_int32), ("chunk_len", C.c_int32)]


class InstanceStatus(C.Structure):
    _fields_ = [("alive", C.c_int32), ("n_requests", C.c_int32), ("blocks_total", C.c_int64),
                ("blocks_used", C.c_int64)]


class ReqStatus(C.Structure):
    _fields_ = [("req_id", C.c_int64), ("prompt_len", C.c_int32), ("n_generated", C.c_int32),
                ("finished", C.c_int32), ("n_blocks", C.c_int32)]


class Timing(C.Structure):
    _fields_ = [("prefill_ms", C.c_double), ("decode_ms", C.c_double), ("prefill_tokens", C.c_int64),
                ("decode_tokens", C.c_int64), ("launches", C.c_int64),
                ("gemm_prefill_ms", C.c_double), ("gemm_prefill_flop", C.c_double), ("gemm_prefill_launches", C.c_int64),
                ("gemm_decode_ms", C.c_double), ("gemm_decode_bytes", C.c_double), ("gemm_decode_launches", C.c_int64),
                ("attn_prefill_ms", C.c_double), ("attn_prefill_flop", C.c_double),
                ("attn_prefill_launches", C.c_int64),
                ("attn_decode_ms", C.c_double), ("attn_decode_bytes", C.c_double), ("attn_decode_launches", C.c_int64),
                ("other_ms", C.c_double), ("other_launches", C.c_int64), ("h2d_bytes", C.c_int64),
                ("d2h_bytes", C.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class ReqState(C.Structure):
    _fields_ = [("req_id", C.c_int64), ("prompt_len", C.c_int32), ("max_new_tokens", C.c_int32),
                ("n_generated", C.c_int32), ("last_token", C.c_int32), ("n_blocks", C.c_int32)]


class MacroConfig(C.Structure):
    _fields_ = [("n_instances", C.c_int32), ("slo_ttft_ns", C.c_int64), ("slo_tpot_ns", C.c_int64),
                ("reserve_tokens", C.c_int32), ("block_tokens", C.c_int32), ("probe_printed", C.c_int32),
                ("cost_a_ns", C.c_int64), ("cost_b_ps", C.c_int64), ("cost_c_ps", C.c_int64),
                ("n_table", C.c_int32), ("table_len", C.POINTER(C.c_int64)), ("table_ns", C.POINTER(C.c_int64)),
                ("total_blocks", C.POINTER(C.c_int64))]


class RouteReq(C.Structure):
    _fields_ = [("req_id", C.c_int64), ("arrival_ns", C.c_int64), ("prompt_len", C.c_int32)]


class SchedReq(C.Structure):
    _fields_ = [("req_id", C.c_int64), ("arrival_ns", C.c_int64), ("prompt_len", C.c_int32),
                ("t_first_ns", C.c_int64), ("n_generated", C.c_int32), ("finished", C.c_int32)]


class SchedStatus(C.Structure):
    _fields_ = [("phase", C.c_int32), ("t_switch_ns", C.c_int64), ("total_blocks", C.c_int64),
                ("alive", C.c_int32)]


class Routed(C.Structure):
    _fields_ = [("req_id", C.c_int64), ("instance", C.c_int32)]


class DesConfig(C.Structure):
    _fields_ = [("cost_d_ns", C.c_int64), ("cost_e_ns", C.c_int64), ("cost_f_ps", C.c_int64),
                ("token_budget", C.c_int32)]


class InstanceHandler(C.Structure):
    _fields_ = [("actor_id", C.c_int64), ("device", C.c_int32), ("tp_size", C.c_int32), ("tp_rank", C.c_int32),
                ("kv_blocks", C.c_int64), ("address", C.c_char * 64)]


P = C.c_void_p
I32, I64, F32 = C.c_int32, C.c_int64, C.c_float
PI32, PI64, PF32 = C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.POINTER(C.c_float)

# name -> (restype, argtypes); every symbol include/*.h declares
SIGNATURES = {
    "ecoserve_nccl_unique_id": (C.c_int, [P]),
    "ecoserve_kv_pool_bytes": (I64, [C.POINTER(ModelShape), I32, I64]),
    "ecoserve_prepared_weight_bytes": (I64, [C.POINTER(ModelShape)]),
    "ecoserve_instance_create": (C.c_int, [C.POINTER(ModelShape), C.POINTER(KVPool), C.POINTER(Weights), P, I32,
                                           I32, P, P, C.POINTER(EngineConfig), C.POINTER(P)]),
    "ecoserve_prefill_phase": (C.c_int, [P, C.POINTER(Request), I32, PI32]),
    "ecoserve_decode_phase": (C.c_int, [P, PI64, I32, I32, PI32, PI32]),
    "ecoserve_hybrid_step": (C.c_int, [P, C.POINTER(Chunk), I32, PI64, I32, PI32, PI32]),
    "ecoserve_release": (C.c_int, [P, PI64, I32]),
    "ecoserve_kv_export": (C.c_int, [P, I64, P, I64, PI32, I32, C.POINTER(ReqState)]),
    "ecoserve_kv_import": (C.c_int, [P, C.POINTER(ReqState), PI32, P]),
    "ecoserve_get_status": (C.c_int, [P, C.POINTER(InstanceStatus), C.POINTER(ReqStatus), I32]),
    "ecoserve_debug_hidden": (C.c_int, [P, I64, I32, PF32]),
    "ecoserve_debug_force_token": (C.c_int, [P, I64, I32]),
    "ecoserve_set_profiling": (C.c_int, [P, I32]),
    "ecoserve_get_timing": (C.c_int, [P, C.POINTER(Timing), I32]),
    "ecoserve_instance_destroy": (None, [P]),
    "ecoserve_last_error": (C.c_char_p, [P]),
    "ecoserve_macro_create": (C.c_int, [C.POINTER(MacroConfig), C.POINTER(P)]),
    "ecoserve_macro_route": (C.c_int, [P, C.POINTER(RouteReq), I64, PI32, PI32, PI32]),
    "ecoserve_macro_check": (C.c_int, [P, I32, C.POINTER(RouteReq), I64, PI32]),
    "ecoserve_macro_defer": (C.c_int, [P, C.POINTER(RouteReq)]),
    "ecoserve_macro_update_status": (C.c_int, [P, I32, C.POINTER(SchedStatus), C.POINTER(SchedReq), I32]),
    "ecoserve_macro_drain_deferred": (C.c_int, [P, I64, C.POINTER(Routed), I32, PI32]),
    "ecoserve_macro_prev_idx": (I32, [P]),
    "ecoserve_macro_predict_prefill_ns": (I64, [P, I32]),
    "ecoserve_macro_destroy": (None, [P]),
    "ecoserve_mitosis_step": (C.c_int, [PI32, PI32, I32, I32, I32, I32, PI32]),
    "ecoserve_handler_serialize": (I32, [C.POINTER(InstanceHandler), C.POINTER(C.c_uint8), I32]),
    "ecoserve_handler_deserialize": (C.c_int, [C.POINTER(C.c_uint8), I32, C.POINTER(InstanceHandler)]),
    "ecoserve_des_run": (C.c_int, [C.POINTER(MacroConfig), C.POINTER(DesConfig), PI64, PI32, PI32, I32, PI32,
                                   PI64, PI64, PI64, PI64, I32, PI32, PI32]),
    "ecoserve_op_gemm": (C.c_int, [P, P, I32, I32, I32, I32, P, I32, P]),
    "ecoserve_op_gemm_swap": (C.c_int, [P, P, I32, I32, I32, I32, P, P, I32, P]),
    "ecoserve_op_gemm_swap_bf16": (C.c_int, [P, P, I32, I32, I32, I32, P, P, P, I32, P]),
    "ecoserve_op_gemm_cluster": (C.c_int, [P, P, I32, I32, I32, I32, P, I32, P]),
    "ecoserve_op_gemm_decode": (C.c_int, [P, P, I32, I32, I32, I32, I32, P, P, I32, P]),
    "ecoserve_op_gemm_decode_balanced": (C.c_int, [P, P, I32, I32, I32, I32, P, P, I32, PI32, P]),
    "ecoserve_op_lm_argmax": (C.c_int, [P, P, I32, I32, I32, P, P, P, P]),
    "ecoserve_op_rmsnorm": (C.c_int, [P, P, P, P, I32, I32, F32, P]),
    "ecoserve_op_attention_prefill": (C.c_int, [P, P, I64, I32, I32, I32, PI32, I32, P, I32, P, P, PI32]),
    "ecoserve_op_attention_prefill_tc": (C.c_int, [P, P, I64, I32, I32, PI32, I32, P, I32, P, P, PI32]),
    "ecoserve_op_attention_decode": (C.c_int, [P, P, I32, I32, I32, P, I32, P, I32, I32, I32, P, P, P, I32]),
    "ecoserve_op_attention_decode_sk": (C.c_int, [P, P, I32, I32, I32, PI32, I32, P, I32, P, P, P, P, P]),
}

_lib = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load the CUDA library (no fallback: raises if it is missing)."""
    global _lib
    if _lib is None:
        path = os.environ.get("ECOSERVE_LIB_AB", path)  # A/B timing of two builds only (tools/)
        if not os.path.exists(path):
            raise ImportError(f"{path} is missing: run `python -m paper_2504_18154_b200.build` "
                              "(the hot path has no CPU fallback)")
        lib = C.CDLL(path)
        ab = "ECOSERVE_LIB_AB" in os.environ
        for name, (res, args) in SIGNATURES.items():
            if ab and not hasattr(lib, name):
                continue  # an older build under A/B timing may lack newer entry points
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(status: int, inst=None) -> None:
    if status != OK:
        msg = ""
        if inst is not None:
            msg = (load().ecoserve_last_error(inst) or b"").decode()
        raise EcoError(status, msg)
