"""ctypes binding of libspecprefill.so (include/specprefill.h), argument marshalling only.

Loading fails loudly if the library is missing: there is no Python or CPU
fallback for any step of the path.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libspecprefill.so")
# development A/B timing only (tools/ab_build.sh): load another build of the same ABI
if os.environ.get("SP_LIB_AB"):
    LIB_PATH = os.environ["SP_LIB_AB"]

SP_OK, SP_EINVAL, SP_EUNSUPPORTED, SP_ECUDA, SP_ENONFINITE, SP_EEMPTY, SP_EWORKSPACE, SP_ETIMEOUT = 0, 1, 2, 3, 5, 6, 7, 8
SP_SCORE_AUTO, SP_SCORE_FUSED, SP_SCORE_SIMT = 0, 1, 2
PLAN_INFO = 10          # entries of sp_score_plan's out array
PLAN_KEYS = ("grid", "jobs_per_request", "token_groups", "unit_groups", "tiles_per_job", "units_per_job",
             "tmem_slots", "stages", "smem_bytes", "hier")
ABI_VERSION = 1


class sp_geom(C.Structure):
    _fields_ = [("B", C.c_int32), ("L", C.c_int32), ("H", C.c_int32), ("Hkv", C.c_int32), ("d", C.c_int32),
                ("R", C.c_int32), ("R_valid", C.c_int32), ("N", C.c_int64), ("scale", C.c_float)]


class sp_layout(C.Structure):
    _fields_ = [("k_b", C.c_int64), ("k_l", C.c_int64), ("k_g", C.c_int64), ("k_i", C.c_int64),
                ("q_b", C.c_int64), ("q_l", C.c_int64), ("q_r", C.c_int64), ("q_h", C.c_int64)]


class sp_select_params(C.Structure):
    _fields_ = [("keep_rate", C.c_double), ("pool_k", C.c_int32), ("chunk", C.c_int32), ("pos0", C.c_int32)]


class sp_paged_k(C.Structure):
    _fields_ = [("cache", C.c_void_p), ("s_l", C.c_int64), ("s_blk", C.c_int64), ("s_tok", C.c_int64),
                ("s_g", C.c_int64), ("num_blocks", C.c_int32), ("block_size", C.c_int32),
                ("block_table", C.c_void_p), ("max_blocks", C.c_int32), ("seq_lens", C.c_void_p)]


class sp_lookahead_k(C.Structure):
    _fields_ = [("K_la", C.c_void_p), ("s_b", C.c_int64), ("s_l", C.c_int64), ("s_g", C.c_int64),
                ("s_j", C.c_int64), ("la_shift", C.c_int32)]


class sp_host_io(C.Structure):
    _fields_ = [("Q", C.c_void_p), ("K", C.c_void_p), ("tokens", C.c_void_p), ("ids", C.c_void_p),
                ("pos", C.c_void_p), ("n_kept", C.c_void_p), ("out_tokens", C.c_void_p),
                ("q_bytes", C.c_size_t), ("k_bytes", C.c_size_t)]


class sp_device_bufs(C.Structure):
    _fields_ = [("Q", C.c_void_p), ("K", C.c_void_p), ("tokens", C.c_void_p), ("importance", C.c_void_p),
                ("ids", C.c_void_p), ("pos", C.c_void_p), ("n_kept", C.c_void_p), ("out_tokens", C.c_void_p),
                ("ws", C.c_void_p), ("ws_bytes", C.c_size_t)]


_P = C.c_void_p
_G = C.POINTER(sp_geom)
_L = C.POINTER(sp_layout)
_S = C.POINTER(sp_select_params)

# name -> (restype, argtypes); every symbol declared in include/specprefill.h
SIGNATURES = {
    "sp_abi_version": (C.c_int, []),
    "sp_status_string": (C.c_char_p, [C.c_int]),
    "sp_kept_chunks": (C.c_int64, [C.c_int64, C.c_double]),
    "sp_check_device_error": (C.c_int, [_P]),
    "sp_device_sm_count": (C.c_int, []),
    "sp_score_workspace_bytes": (C.c_size_t, [_G, C.c_int]),
    "sp_score": (C.c_int, [_P, _P, _G, _L, _P, _P, C.c_size_t, _P]),
    "sp_score_ex": (C.c_int, [_P, _P, _G, _L, _P, _P, C.c_size_t, C.c_int, _P]),
    "sp_score_plan": (C.c_int, [_G, C.POINTER(C.c_int64)]),
    "sp_score_tune": (C.c_int, [_P, _P, _G, _L, C.POINTER(C.c_int64), C.POINTER(C.c_float), _P]),
    "sp_score_e4m3_tune": (C.c_int, [_P, _P, C.c_float, C.c_float, _G, _L, C.POINTER(C.c_int64),
                                     C.POINTER(C.c_float), _P]),
    "sp_score_set_plan": (C.c_int, [_G, C.c_int32, C.c_int32, C.c_int32]),
    "sp_trace_enable": (C.c_int, [_P, C.c_int64]),
    "sp_score_split_workspace_bytes": (C.c_size_t, [_G]),
    "sp_score_stats": (C.c_int, [_P, _P, _G, _L, _P, _P, C.c_size_t, _P]),
    "sp_stats_combine": (C.c_int, [_P, C.c_int32, C.c_int64, _P, _P]),
    "sp_score_finish": (C.c_int, [_P, _P, _G, _L, _P, _P, _P, C.c_size_t, _P]),
    "sp_score_acc": (C.c_int, [_P, _P, _G, _L, _P, _P, C.c_size_t, _P]),
    "sp_acc_importance": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int64, _P, _P]),
    "sp_score_peer_buffer_bytes": (C.c_size_t, [_G, C.c_int32, C.c_int32]),
    "sp_score_peer_workspace_bytes": (C.c_size_t, [_G, C.c_int32, C.c_int32]),
    "sp_score_peer_plan": (C.c_int, [_G, C.c_int32, C.c_int32, C.POINTER(C.c_int64)]),
    "sp_score_peer": (C.c_int, [_P, _P, _G, _L, C.c_int32, C.c_int32, C.POINTER(C.c_void_p), C.c_int32, _P, _P,
                                C.c_size_t, _P]),
    "sp_score_e4m3_workspace_bytes": (C.c_size_t, [_G]),
    "sp_score_e4m3_plan": (C.c_int, [_G, C.POINTER(C.c_int64)]),
    "sp_score_e4m3": (C.c_int, [_P, _P, C.c_float, C.c_float, _G, _L, _P, _P, C.c_size_t, _P]),
    "sp_score_lookahead_workspace_bytes": (C.c_size_t, [_G]),
    "sp_score_lookahead": (C.c_int, [_P, _P, C.POINTER(sp_lookahead_k), _G, _L, _P, _P, C.c_size_t, _P]),
    "sp_score_paged_workspace_bytes": (C.c_size_t, [_G]),
    "sp_score_paged": (C.c_int, [_P, C.POINTER(sp_paged_k), _G, _L, _P, _P, C.c_size_t, _P]),
    "sp_score_paged_e4m3": (C.c_int, [_P, C.POINTER(sp_paged_k), C.c_float, C.c_float, _G, _L, _P, _P, C.c_size_t,
                                      _P]),
    "sp_select_ragged": (C.c_int, [_P, _P, _P, C.c_int32, C.c_int64, _S, _P, _P, _P, _P, _P, C.c_size_t, _P]),
    "sp_select_workspace_bytes": (C.c_size_t, [C.c_int32, C.c_int64, _S]),
    "sp_select": (C.c_int, [_P, C.c_int32, C.c_int64, _S, _P, _P, _P, _P, C.c_size_t, _P]),
    "sp_select_gather": (C.c_int, [_P, _P, C.c_int32, C.c_int64, _S, _P, _P, _P, _P, _P, C.c_size_t, _P]),
    "sp_gather": (C.c_int, [_P, _P, _P, C.c_int32, C.c_int64, _P, _P]),
    "sp_seq_candidate_count": (C.c_int64, [C.c_int64, C.c_int32, _S]),
    "sp_seq_select_workspace_bytes": (C.c_size_t, [C.c_int32, C.c_int64, C.c_int32, _S]),
    "sp_seq_edges": (C.c_int, [_P, C.c_int32, C.c_int64, C.c_int32, _S, _P, _P]),
    "sp_seq_candidates": (C.c_int, [_P, _P, C.c_int32, C.c_int32, C.c_int32, C.c_int64, _S, _P, _P, C.c_size_t, _P]),
    "sp_seq_merge": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int64, _S, _P, _P, _P, _P, _P, _P, C.c_size_t, _P]),
    "sp_score_select_workspace_bytes": (C.c_size_t, [_G, _S]),
    "sp_score_select": (C.c_int, [_P, _P, _G, _L, _S, _P, _P, _P, _P, _P, _P, _P, C.c_size_t, _P]),
    "sp_score_chunks": (C.c_int, [_P, _P, _G, _L, C.c_int32, C.c_int32, _P, _P, _P, C.c_size_t, _P]),
    "sp_run_workspace_bytes": (C.c_size_t, [_G, _S]),
    "sp_run_host": (C.c_int, [C.POINTER(sp_host_io), C.POINTER(sp_device_bufs), _G, _L, _S, _P]),
}

_lib = None


class SpError(RuntimeError):
    def __init__(self, code: int, where: str):
        self.code = code
        msg = lib().sp_status_string(code).decode() if code >= 0 else "unknown"
        super().__init__(f"{where}: {msg}")


def lib():
    """Load libspecprefill.so (once).  Raises if it is missing: build it with
    ``python -c 'import __graft_entry__ as g; g.build()'``."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: the CUDA extension is required (no CPU fallback); "
                              "run __graft_entry__.build()")
        h = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            if os.environ.get("SP_LIB_AB") and not hasattr(h, name):
                continue                       # A/B timing of an older build (tools/ab_build.sh)
            f = getattr(h, name)
            f.restype = res
            f.argtypes = args
        if h.sp_abi_version() != ABI_VERSION:
            raise ImportError("libspecprefill.so ABI version mismatch")
        _lib = h
    return _lib


def check(code: int, where: str):
    if code != SP_OK:
        raise SpError(code, where)
