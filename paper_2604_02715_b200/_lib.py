"""ctypes binding of libxpgb.so (C ABI declared in include/xpgb.h).

The library is built in-tree (``python -m paper_2604_02715_b200.build``).  There
is no fallback: if the shared object is missing or cannot be loaded, importing
anything that needs it raises ``XpgError`` immediately.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import XpgError, raise_for_status

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("XPGB_LIB_PATH") or os.path.join(_HERE, "libxpgb.so")  # override: A/B builds

# ---- enums (mirror include/xpgb.h)
POOL_RING = 0
POOL_RESIDENT = 1
EV_RECYCLE, EV_LOAD_START, EV_LOAD_DONE, EV_COMPUTE_START, EV_COMPUTE_DONE, EV_RUN_BEGIN = range(6)
EVENT_NAMES = {
    EV_RECYCLE: "recycle",
    EV_LOAD_START: "load-start",
    EV_LOAD_DONE: "load-done",
    EV_COMPUTE_START: "compute-start",
    EV_COMPUTE_DONE: "compute-done",
    EV_RUN_BEGIN: "run-begin",
}


class Spec(C.Structure):
    _fields_ = [("num_layers", C.c_int32), ("experts_per_layer", C.c_int32), ("hidden_dim", C.c_int32),
                ("intermediate_dim", C.c_int32)]


class Record(C.Structure):
    _fields_ = [("t", C.c_int32), ("event", C.c_int32), ("iteration", C.c_int32), ("layer", C.c_int32),
                ("kind", C.c_int32), ("target_iteration", C.c_int32), ("target_layer", C.c_int32),
                ("group", C.c_int32), ("wall_ns", C.c_int64)]


class RunOpts(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("tokens", C.c_int32), ("top_k", C.c_int32), ("sequential", C.c_int32),
                ("router_seed", C.c_uint64), ("sabotage_iteration", C.c_int32), ("sabotage_layer", C.c_int32),
                ("fetch_delay_s", C.POINTER(C.c_float)), ("compute_delay_s", C.POINTER(C.c_float)),
                ("log_enable", C.c_int32), ("profile", C.c_int32), ("fresh_inputs", C.c_int32)]


class Report(C.Structure):
    _fields_ = [("stall_ns", C.c_int64), ("war_wait_ns", C.c_int64), ("elapsed_ns", C.c_int64),
                ("arena_peak_bytes", C.c_int64), ("h2d_bytes", C.c_int64), ("d2d_bytes", C.c_int64),
                ("copy_busy_ns", C.c_int64 * 2), ("page_fault", C.c_int32), ("n_records", C.c_int32),
                ("kern_gate_up_ns", C.c_double), ("kern_down_ns", C.c_double), ("kern_aux_ns", C.c_double),
                ("gate_up_bytes", C.c_int64), ("down_bytes", C.c_int64), ("down_splits", C.c_int32),
                ("active_experts", C.c_int32), ("decoded_bytes", C.c_int64)]


class KernelTimes(C.Structure):
    _fields_ = [("route_ns", C.c_double), ("plan_ns", C.c_double), ("gather_ns", C.c_double),
                ("gate_up_ns", C.c_double), ("down_ns", C.c_double), ("combine_ns", C.c_double),
                ("gate_up_bytes", C.c_int64), ("down_bytes", C.c_int64), ("down_splits", C.c_int32),
                ("n_units_gate_up", C.c_int32), ("n_units_down", C.c_int32)]


class EpPlanBufs(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("src_rows", "dst_rank", "dst_row", "ret_index", "c_rank", "c_row",
                                           "to_arrival", "from_arrival", "offsets", "counts")]


_P = C.c_void_p
_I = C.c_int32
_U64 = C.c_uint64
# name -> argtypes (all return int status unless listed in _RESTYPES)
_SIGS = {
    "xpgb_abi_version": [],
    "xpgb_last_error": [],
    "xpgb_kernel_launches": [],
    "xpgb_create": [C.POINTER(Spec), _I, _I, _I, C.POINTER(_P)],
    "xpgb_create_shard": [C.POINTER(Spec), _I, _I, _I, _I, _I, C.POINTER(_P)],
    "xpgb_destroy": [_P],
    "xpgb_sync": [_P],
    "xpgb_pinned_alloc": [_U64, C.POINTER(_P)],
    "xpgb_pinned_free": [_P],
    "xpgb_host_pool_alloc": [_P, C.POINTER(_P), C.POINTER(_U64)],
    "xpgb_host_pool_register": [_P, _P, _U64],
    "xpgb_set_placement": [_P, C.POINTER(C.c_uint8)],
    "xpgb_fetch": [_P, _I, _I, _I, _P, _U64, _P],
    "xpgb_pt_map": [_P, _I, _I, _I, C.POINTER(_I)],
    "xpgb_pt_mark_resident": [_P, _I, _I, _I],
    "xpgb_pt_unmap": [_P, _I, _I, _I],
    "xpgb_pt_state": [_P, _I, _I, _I, C.POINTER(_I)],
    "xpgb_pt_block": [_P, _I, _I, _I, C.POINTER(_I)],
    "xpgb_pt_block_ptr": [_P, _I, _I, C.POINTER(_P), C.POINTER(_U64)],
    "xpgb_pt_loading_view": [_P, _I, _I, _I, C.POINTER(_P), C.POINTER(_U64)],
    "xpgb_pt_read": [_P, _I, _I, _I, _P, _U64],
    "xpgb_pt_peak_bytes": [_P, C.POINTER(_U64)],
    "xpgb_pt_pool_bytes": [_P, C.POINTER(_U64)],
    "xpgb_pt_check_consistency": [_P],
    "xpgb_pt_trace_enable": [_P, _I],
    "xpgb_pt_trace_get": [_P, C.c_char_p, _U64, C.POINTER(_U64)],
    "xpgb_make_resident": [_P],
    "xpgb_route": [_U64, _I, _I, _I, _I, _I, _P, _P],
    "xpgb_layer_forward": [_P, _I, _P, _P, _I, _I, _U64, _P],
    "xpgb_fault_get": [_P, C.POINTER(_I), C.c_char_p, _U64],
    "xpgb_fault_clear": [_P],
    "xpgb_run": [_P, C.POINTER(RunOpts), _P, _P, C.POINTER(Report)],
    "xpgb_session_begin": [_P, C.POINTER(RunOpts), _P],
    "xpgb_session_materialize": [_P, _I],
    "xpgb_session_acquire": [_P, _I, _P],
    "xpgb_session_compute": [_P, _I],
    "xpgb_session_run_steps": [_P, _I, _I, _P],
    "xpgb_session_release": [_P, _I, _P],
    "xpgb_session_end": [_P, C.POINTER(Report)],
    "xpgb_session_abort": [_P],
    "xpgb_session_info": [_P, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_void_p)],
    "xpgb_log_get": [_P, C.POINTER(Record), _I, C.POINTER(_I)],
    "xpgb_set_expert_shard": [_P, _I, _I],
    "xpgb_set_shared": [_P, _P, _U64, _I],
    "xpgb_host_register": [_P, _U64, _I],
    "xpgb_host_unregister": [_P],
    "xpgb_set_ring_experts": [_P, _I],
    "xpgb_set_ring_depth": [_P, _I],
    "xpgb_set_fused_decode": [_P, _I],
    "xpgb_set_activation_planes": [_P, _I],
    "xpgb_set_device_format": [_P, _I],
    "xpgb_set_device_formats": [_P, C.POINTER(C.c_uint8)],
    "xpgb_set_host_staging": [_P, _I],
    "xpgb_set_hazard_checks": [_P, _I, _I, _I],
    "xpgb_set_stage_buffers": [_P, _I],
    "xpgb_decode_stats": [_P, _P, _P, _P],
    "xpgb_fused_stats": [_P, _P, _P, _P],
    "xpgb_ep_window_alloc": [C.c_uint64, _P, _P],
    "xpgb_ep_window_open": [_P, _P],
    "xpgb_ep_window_close": [_P],
    "xpgb_ep_window_free": [_P],
    "xpgb_ep_scatter_rows": [_P, _P, _P, _P, _I, _P, _I, _I, C.c_int64, _P, _P, _I, _I, _I, _P, _P, _P],
    "xpgb_ep_wait": [_P, _I, _I, _P, _P],
    "xpgb_ep_reduce_scatter": [_P, _P, _P, _I, _P, _P, _P, _I, _I, _I, _P, _P],
    "xpgb_fault_ptr": [_P, C.POINTER(_P)],
    "xpgb_fault_set": [_P, C.c_int64],
    "xpgb_ep_plan_scratch_words": [_I, _I, _I],
    "xpgb_ep_plan": [_P, _I, _I, _I, _I, _I, _P, C.POINTER(EpPlanBufs), _P],
    "xpgb_set_shared_tokens": [_P, _I, _I],
    "xpgb_shared_forward": [_P, _I, _P, _P, _I, _P],
    "xpgb_experts_forward": [_P, _I, _P, C.c_int64, _P, _I, _P, _P],
    "xpgb_experts_forward_range": [_P, _I, _P, C.c_int64, _P, _I, _I, _I, _I, _P, _P],
    "xpgb_session_step": [_P, _I, C.POINTER(C.c_int32)],
    "xpgb_combine_rows": [_P, _P, _I, _I, _I, _I, _P, _P],
    "xpgb_codec_histogram": [_P, _U64, C.POINTER(_U64), _I],
    "xpgb_codec_encode": [_P, _U64, C.POINTER(C.c_uint8), _P, _P, _U64, C.POINTER(_U64), C.POINTER(_U64),
                          C.POINTER(C.c_uint32), _I],
    "xpgb_codec_pack": [_P, _I, C.POINTER(_U64), C.POINTER(C.c_uint8), _I, _I, C.POINTER(C.c_int32), _P, _U64,
                        C.POINTER(_U64),
                        C.POINTER(_U64), C.POINTER(_U64), C.POINTER(_U64)],
    "xpgb_codec_record_bytes": [_U64, _U64, _I],
    "xpgb_codec_index": [_P, _U64, _U64, C.POINTER(C.c_uint8), _I, C.POINTER(C.c_uint32), C.POINTER(_U64)],
    "xpgb_codec_decode": [_P, _U64, _U64, _I, C.POINTER(C.c_uint8), _P, _P],
    "xpgb_fx4_scratch_bytes": [_U64],
    "xpgb_fx4_measure": [_P, _U64, _P, C.POINTER(C.c_int32), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), _P],
    "xpgb_fx4_encode": [_P, _U64, _I, _P, _P, _P],
    "xpgb_fx4_decode": [_P, _U64, _I, _P, _P],
    "xpgb_set_codec": [_P, _P, _U64, C.POINTER(_U64), C.POINTER(_U64), C.POINTER(C.c_uint8), _I, _I],
    "xpgb_set_pinned": [_P, C.POINTER(C.c_uint8)],
    "xpgb_hbm_bytes": [_P, C.POINTER(_U64), C.POINTER(_U64), C.POINTER(_U64)],
    "xpgb_profile_layer": [_P, _I, _P, _P, _I, _I, _U64, _I, C.POINTER(KernelTimes)],
}
_RESTYPES = {"xpgb_last_error": C.c_char_p, "xpgb_kernel_launches": C.c_int64, "xpgb_codec_record_bytes": C.c_uint64,
             "xpgb_ep_plan_scratch_words": C.c_int64, "xpgb_fx4_scratch_bytes": C.c_uint64}

# every symbol declared in include/xpgb.h (tests check the export table against this)
DECLARED = tuple(_SIGS)

_lib = None


def lib():
    """Load libxpgb.so once; raise XpgError (no fallback) if it is unavailable."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise XpgError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2604_02715_b200.build` "
            "(the B200 path has no CPU fallback)"
        )
    try:
        handle = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    except OSError as exc:  # pragma: no cover - environment dependent
        raise XpgError(f"cannot load {LIB_PATH}: {exc}") from exc
    for name, args in _SIGS.items():
        fn = getattr(handle, name)
        fn.argtypes = args
        fn.restype = _RESTYPES.get(name, C.c_int)
    if handle.xpgb_abi_version() != 1:
        raise XpgError("libxpgb ABI version mismatch")
    _lib = handle
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        msg = lib().xpgb_last_error()
        raise_for_status(rc, msg.decode() if msg else "")


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))
