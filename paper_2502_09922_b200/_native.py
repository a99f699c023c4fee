"""ctypes binding of the in-tree C-ABI library ``liblambdapipe.so``.

The product path has no CPU fallback: if the library is missing or fails to
load, :func:`lib` raises and every device entry point fails loudly.  Argument
types are declared from ``include/lambdapipe.h``; :func:`check` maps a
negative status to :class:`NativeError` carrying ``lp_last_error()``.
"""

from __future__ import annotations

import ctypes as C
import os
import re

from .errors import NativeError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liblambdapipe.so")
HEADER = os.path.join(HERE, "..", "include", "lambdapipe.h")

_vp, _i32, _i64, _u32, _u64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.c_uint64
_P = C.POINTER

# name -> argtypes (restype is int unless listed in _RESTYPE)
SIGNATURES = {
    "lp_version": [],
    "lp_last_error": [],
    "lp_device_count": [_P(C.c_int)],
    "lp_set_device": [C.c_int],
    "lp_set_pdl": [C.c_int],
    "lp_sync_device": [C.c_int],
    "lp_enable_peer": [C.c_int, C.c_int],
    "lp_malloc": [C.c_int, _i64, _P(_vp)],
    "lp_free": [C.c_int, _vp],
    "lp_memset": [_vp, C.c_int, _i64, _vp],
    "lp_memcpy": [_vp, _vp, _i64, _vp],
    "lp_ipc_get": [_vp, _vp],
    "lp_ipc_open": [C.c_int, _vp, _P(_vp)],
    "lp_ipc_close": [_vp],
    "lp_host_register": [_vp, _i64, _P(_vp)],
    "lp_host_unregister": [_vp],
    "lp_stream_create": [C.c_int, _P(_vp)],
    "lp_stream_destroy": [_vp],
    "lp_stream_sync": [_vp],
    "lp_event_create": [_P(_vp)],
    "lp_event_destroy": [_vp],
    "lp_event_record": [_vp, _vp],
    "lp_event_elapsed_ms": [_vp, _vp, _P(C.c_float)],
    "lp_fill_tensors": [_vp, C.c_int, _P(_i64), _P(_i64), _P(_i32), _P(_i32), _u64, _vp],
    "lp_block_checksums": [_vp, C.c_int, _P(_i64), _P(_i64), _P(_u64), _vp],
    "lp_mc_create": [_P(_vp), C.c_int, C.c_int, _P(_i64), _P(_i64), _i64],
    "lp_mc_create_tiled": [_P(_vp), C.c_int, C.c_int, _P(_i64), _P(_i64), _P(_i64)],
    "lp_mc_destroy": [_vp],
    "lp_mc_signal_bytes": [_vp, _P(_i64)],
    "lp_mc_set_node": [_vp, C.c_int, C.c_int, _vp, _vp, _vp],
    "lp_mc_set_schedule": [_vp, _P(_i32), C.c_int, _P(_i32), C.c_int],
    "lp_mc_run": [_vp, _P(_i32), C.c_int, _u32, C.c_int, C.c_int, _vp],
    "lp_mc_status": [_vp, _vp, _P(C.c_int)],
    "lp_mc_configure": [_vp, C.c_int, C.c_int, C.c_int, _i64, C.c_int],
    "lp_mc_run_ce": [_vp, C.c_int, _u32, C.c_int, _P(_vp), _P(_vp)],
    "lp_mc_landing_events": [_vp, C.c_int, _u32, _vp, _P(_vp)],
    "lp_mc_run_host_dma": [_vp, C.c_int, _u32, C.c_int, _P(_vp), _P(_vp)],
    "lp_mc_node_ops": [_vp, C.c_int, _P(C.c_int), _P(C.c_int)],
    "lp_mc_verify": [_vp, C.c_int, _u32, C.c_int, _vp, _vp],
    "lp_mc_set_option": [_vp, C.c_char_p, _i64],
    "lp_mc_reset_signals": [_vp, C.c_int, _vp],
    "lp_mc_arrivals": [_vp, C.c_int, _P(_u64)],
    "lp_mc_block_complete": [_vp, C.c_int, _u32, _P(_i32)],
    "lp_gemm_bf16": [_vp, _i64, _i64, _vp, _i64, _vp, _i64, C.c_int, C.c_int, _vp],
    "lp_gemm_swiglu": [_vp, _vp, _i64, _i64, _vp, _i64, _vp, _i64, _vp],
    "lp_embed": [_vp, _i64, _vp, _i64, _vp, _vp],
    "lp_rmsnorm": [_vp, _vp, _i64, _i64, C.c_float, _vp, _vp],
    "lp_rmsnorm_zero": [_vp, _vp, _i64, _i64, C.c_float, _vp, _vp, _i64, _vp],
    "lp_rope_kv": [_vp, _i64, C.c_int, C.c_int, C.c_int, _vp, _vp, C.c_float, _vp, _vp, _vp, _i64, _vp],
    "lp_attention": [_vp, _vp, _vp, _vp, _vp, _i64, C.c_int, C.c_int, C.c_int, _i64, C.c_float, _vp, _vp],
    "lp_argmax": [_vp, _i64, _i64, _vp, _vp, _vp],
    "lp_handoff": [_vp, _vp, _i64, _vp, _u32, _vp, _vp],
}
_RESTYPE = {"lp_last_error": C.c_char_p}

_LIB = None


def header_symbols() -> list:
    """Every ``lp_*`` function declared in include/lambdapipe.h."""
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(lp_\w+)\s*\(", text, re.M)))


def lib():
    """Load (once) and return the library; raise if it is absent."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise NativeError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                          "(there is no CPU fallback for the CUDA path)")
    handle = C.CDLL(LIB_PATH)
    for name, args in SIGNATURES.items():
        fn = getattr(handle, name)
        fn.argtypes = args
        fn.restype = _RESTYPE.get(name, C.c_int)
    _LIB = handle
    return _LIB


def check(status: int, what: str = "") -> None:
    if status < 0:
        msg = lib().lp_last_error().decode(errors="replace")
        raise NativeError(f"{what or 'lambdapipe'} failed ({status}): {msg}")


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args), name)


def i64_array(vals):
    arr = (_i64 * len(vals))(*vals)
    return arr


def i32_array(vals):
    return (_i32 * len(vals))(*vals)


def stream_ptr(stream) -> int:
    """cudaStream_t of a torch stream (or 0)."""
    if stream is None:
        return 0
    return int(stream.cuda_stream)
