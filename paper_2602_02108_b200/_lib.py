"""ctypes binding of liboomb.so (include/oomb.h).

The product path has no fallback: if the library is missing or cannot be
loaded, importing the operator modules raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

from .errors import raise_for_status

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "liboomb.so")
COMM_LIB_PATH = os.path.join(PKG, "liboomb_comm.so")

I32P = C.POINTER(C.c_int32)


class OombConfig(C.Structure):
    _fields_ = [
        ("n_layers", C.c_int), ("n_q_heads", C.c_int), ("n_kv_heads", C.c_int), ("head_dim", C.c_int),
        ("chunk_size", C.c_int), ("page_size", C.c_int), ("retrieval_budget", C.c_int), ("local_window", C.c_int),
        ("score_scale", C.c_int), ("dtype", C.c_int), ("max_tokens", C.c_int64),
        ("device_capacity_pages", C.c_int64), ("page_owner_stride", C.c_int), ("page_owner_rank", C.c_int),
    ]


class OombMemoryReport(C.Structure):
    _fields_ = [
        ("device_bytes", C.c_uint64), ("host_bytes", C.c_uint64), ("grad_bytes", C.c_uint64), ("pages", C.c_int64),
        ("reallocs", C.c_int64), ("copied_bytes", C.c_uint64), ("arena_blocks", C.c_int64), ("free_list", C.c_int64),
    ]


VP = C.c_void_p
I = C.c_int
I64 = C.c_int64

# name -> argtypes (all return int status unless listed in _RESTYPE)
_PROTOS = {
    "oomb_last_error": [],
    "oomb_version": [],
    "oomb_kernel_launches": [],
    "oomb_pool_create": [C.POINTER(OombConfig), I, C.POINTER(VP)],
    "oomb_pool_destroy": [VP],
    "oomb_pool_reset": [VP, VP],
    "oomb_zero_grad_pages": [VP, VP],
    "oomb_memory_report_get": [VP, C.POINTER(OombMemoryReport)],
    "oomb_check_device_errors": [VP],
    "oomb_append_chunk": [VP, I, VP, VP, I64, VP, C.POINTER(I64), C.POINTER(I64)],
    "oomb_append_chunk_rope": [VP, I, VP, VP, I64, C.c_float, VP, C.POINTER(I64), C.POINTER(I64)],
    "oomb_rope": [VP, I64, I, I, I64, C.c_float, I, I, I, VP, VP],
    "oomb_n_pages": [VP, I, C.POINTER(I)],
    "oomb_filled": [VP, I, C.POINTER(I64)],
    "oomb_page_table_get": [VP, I, VP],
    "oomb_device_slots_get": [VP, I, VP],
    "oomb_page_mean_keys": [VP, I, I, VP, VP, C.POINTER(I)],
    "oomb_kavg_raw": [VP, I, VP, VP, VP],
    "oomb_gather_pages": [VP, I, VP, I, I, VP, VP, VP, VP],
    "oomb_scatter_add_grads": [VP, I, VP, I, VP, VP, VP],
    "oomb_set_tier": [VP, I, I, I],
    "oomb_get_tier": [VP, I, I, C.POINTER(I)],
    "oomb_set_residency_enforced": [VP, I],
    "oomb_grads_allocated": [VP, I, I, C.POINTER(I)],
    "oomb_selection_create": [VP, I, I, C.POINTER(VP)],
    "oomb_selection_destroy": [VP],
    "oomb_selection_set_host": [VP, VP, VP, I, VP],
    "oomb_selection_get_host": [VP, VP, VP, C.POINTER(I), C.POINTER(I)],
    "oomb_selection_device": [VP, C.POINTER(VP), C.POINTER(VP), C.POINTER(I)],
    "oomb_select_all": [VP, I, I, VP],
    "oomb_select_recent": [VP, I, I, I, VP],
    "oomb_select_topk": [VP, VP, I, I, I, VP],
    "oomb_selection_filter_owned": [VP, VP, VP, VP],
    "oomb_page_owner": [VP, C.POINTER(I), C.POINTER(I)],
    "oomb_score_pages": [VP, I64, I, I, VP, I64, I, I, I, I, VP, VP],
    "oomb_select_pages_topk": [VP, I, VP, I64, I, VP, VP, VP],
    "oomb_attn_forward": [VP, I, VP, I64, VP, VP, VP, VP, VP, VP],
    "oomb_attn_backward": [VP, I, VP, VP, I64, VP, VP, VP, VP, VP, VP, VP, VP, VP],
    "oomb_attn_forward_ex": [VP, I, VP, I64, VP, VP, VP, VP, VP, I, VP],
    "oomb_attn_backward_ex": [VP, I, VP, VP, I64, VP, VP, VP, VP, VP, VP, VP, VP, I, VP],
    "oomb_lse_merge": [VP, VP, I, I64, I, I, VP, VP, VP],
    "oomb_set_kernel_policy": [VP, I],
    "oomb_pagetable_create": [I, I, I, I, I, I, C.POINTER(VP)],
    "oomb_pagetable_destroy": [VP],
    "oomb_pagetable_append": [VP, I, I64, C.POINTER(I64), C.POINTER(I64)],
    "oomb_pagetable_scatter": [VP, I, VP, I],
    "oomb_pagetable_reset": [VP],
    "oomb_pagetable_n_pages": [VP, I, C.POINTER(I)],
    "oomb_pagetable_get": [VP, I, VP],
    "oomb_pagetable_set_tier": [VP, I, I, I],
    "oomb_pagetable_memory_report": [VP, C.POINTER(OombMemoryReport)],
    "oomb_debug_tc_gemm": [I, VP, VP, VP, I, I, I, VP],
    "oomb_accumulate_grad_pages": [VP, I, VP, I, VP, VP, VP],
    "oomb_profile_enable": [VP, I],
    "oomb_profile_collect": [VP, VP, VP, I],
    "oomb_tier_create_sim": [VP, VP, C.POINTER(VP)],
    "oomb_tier_create": [VP, VP, VP, C.POINTER(VP)],
    "oomb_tier_destroy": [VP],
    "oomb_tier_begin_phase": [VP, I],
    "oomb_tier_set_prefetch_headroom": [VP, I64],
    "oomb_tier_on_pages_appended": [VP, I, I64, I64],
    "oomb_tier_on_grads_scattered": [VP, I, VP, I],
    "oomb_tier_fetch_async": [VP, I, VP, I, I, I, C.POINTER(I64)],
    "oomb_tier_wait": [VP, I64],
    "oomb_tier_record_access": [VP, I, VP, I, I],
    "oomb_tier_advance_compute": [VP, C.c_double, I, I],
    "oomb_tier_end_layer_use": [VP, I, VP, I],
    "oomb_tier_release_all": [VP],
    "oomb_tier_restore_all": [VP],
    "oomb_tier_stats": [VP, VP],
    "oomb_tier_log": [VP, VP, I64, C.POINTER(I64)],
    "oomb_tier_moved_bytes": [VP, C.POINTER(I64), C.POINTER(I64)],
    "oomb_validate_schedule": [VP, I64, C.c_double, VP, C.POINTER(I), VP, VP, I64],
    "oomb_score_pages_partial": [VP, I, VP, I64, I, VP, VP],
    "oomb_vote_reduce": [VP, I, I64, I64, VP, VP],
    "oomb_attn_join_dq": [VP, VP],
    "oomb_attn_backward_readback": [VP, I, VP, VP, I64, VP, VP, VP, VP, VP, VP, VP, VP, I, I64, VP],
    "oomb_layer_step": [VP, I, I, I, VP, I, VP, VP, VP, I, VP, VP, VP, VP, VP, I64, I, VP],
    "oomb_layer_stats": [VP, VP, I64, C.POINTER(I64)],
    "oomb_accumulate_grad_pages_rope": [VP, I, VP, I, VP, VP, I64, C.c_float, VP],
}
_RESTYPE = {"oomb_last_error": C.c_char_p, "oomb_kernel_launches": C.c_int64}

_lib = None


def lib() -> C.CDLL:
    """Load liboomb.so once; raise loudly when it is absent (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} not found: build it with `python -m paper_2602_02108_b200.build` "
                "(the OOMB operators have no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, args in _PROTOS.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = _RESTYPE.get(name, C.c_int)
        _lib = L
    return _lib


def call(name: str, *args) -> None:
    L = lib()
    rc = getattr(L, name)(*args)
    if rc != 0:
        raise_for_status(rc, L.oomb_last_error().decode(errors="replace"))


def kernel_launches() -> int:
    return int(lib().oomb_kernel_launches())


def exported_symbols() -> list[str]:
    return list(_PROTOS)


# liboomb_comm.so (include/oomb_comm.h): NCCL exchange steps of the sharded path
_COMM_PROTOS = {
    "oomb_comm_last_error": [],
    "oomb_comm_get_unique_id": [VP],
    "oomb_comm_init": [VP, I, I, I, VP],
    "oomb_comm_destroy": [VP],
    "oomb_comm_rank": [VP, VP, VP],
    "oomb_vote_allgather": [VP, VP, I, I64, I64, VP, VP],
    "oomb_lse_merge_allgather": [VP, VP, VP, I64, I, I, VP, VP, VP],
    "oomb_dq_reduce": [VP, VP, I64, VP, VP],
    "oomb_allreduce_ordered": [VP, VP, I64, VP, VP],
    "oomb_lse_merge_ordered": [VP, VP, VP, I64, I, I, VP, VP, VP],
    "oomb_comm_bytes": [I, I, I64, I64, C.POINTER(I64), C.POINTER(I64)],
}
_comm = None


def comm_lib() -> C.CDLL:
    """Load liboomb_comm.so once (it pulls in liboomb.so and NCCL); raise loudly when absent."""
    global _comm
    if _comm is None:
        lib()
        if not os.path.exists(COMM_LIB_PATH):
            raise ImportError(f"{COMM_LIB_PATH} not found: build it with `python -m paper_2602_02108_b200.build`")
        L = C.CDLL(COMM_LIB_PATH)
        for name, args in _COMM_PROTOS.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_char_p if name == "oomb_comm_last_error" else C.c_int
        _comm = L
    return _comm


def comm_call(name: str, *args) -> None:
    L = comm_lib()
    rc = getattr(L, name)(*args)
    if rc != 0:
        raise_for_status(rc, L.oomb_comm_last_error().decode(errors="replace"))


def comm_exported_symbols() -> list[str]:
    return list(_COMM_PROTOS)
