"""ctypes binding of the C-ABI library (include/star_attn.h -> libstar_attn.so).

The library is built in-tree by `python __graft_entry__.py build` (or `make -C
paper_2411_17116_b200/csrc`).  There is no fallback: if the shared object is
missing or a call fails, the caller gets an exception.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import c_double, c_float, c_int, c_int64, c_uint64, c_void_p, POINTER

from .errors import ConfigError, DeviceError, DomainError, ShapeError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libstar_attn.so")

STAR_OK, STAR_ESHAPE, STAR_EDOMAIN, STAR_ECONFIG, STAR_ECUDA, STAR_ENOTSUP = 0, -1, -2, -3, -4, -5
STAR_F32, STAR_BF16 = 0, 1

# name -> (restype, argtypes); mirrors include/star_attn.h one to one
SIGNATURES = {
    "star_version": (c_int, []),
    "star_last_error": (ctypes.c_char_p, []),
    "star_prng_fill": (c_int, [c_void_p, c_int, c_int64, c_uint64, c_uint64, c_double, c_void_p]),
    "star_rope": (c_int, [c_void_p, c_void_p, c_int, c_int64, c_int, c_int, c_int64, c_int64,
                          c_void_p, c_double, c_void_p]),
    "star_rope_qkv": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int64, c_int, c_int, c_int,
                              c_int64, c_int64, c_void_p, c_void_p, c_int64, c_int64, c_void_p,
                              c_double, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_void_p]),
    "star_kv_append": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_int,
                               c_int, c_int64, c_int64, c_void_p, c_int64, c_void_p, c_double,
                               c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int, c_void_p,
                               c_int64, c_int64, c_void_p]),
    "star_rope_table": (c_int, [c_void_p, c_int64, c_int64, c_int, c_double, c_void_p]),
    "star_phase2_decode": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int64, c_int64, c_void_p,
                                   c_double, c_void_p, c_int64, c_int64, c_void_p, c_int, c_int,
                                   c_int, c_int,
                                   c_void_p, c_void_p, c_int64, c_void_p, c_int, c_int, c_void_p,
                                   c_int64, c_void_p, c_void_p, c_int, c_void_p, c_void_p]),
    "star_phase2_decode_exchange": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int64, c_int64,
                                            c_void_p, c_double, c_void_p, c_int64, c_int64,
                                            c_void_p, c_int,
                                            c_int, c_int, c_int, c_void_p, c_void_p, c_int64,
                                            c_void_p, c_int, c_int, c_void_p, c_int64, c_void_p,
                                            c_void_p, c_int, c_void_p, c_void_p, c_int, c_int64,
                                            c_int, c_int, c_void_p]),
    "star_decode_advance": (c_int, [c_void_p, c_int, c_int, c_void_p, c_int, c_int, c_void_p,
                                    c_void_p, c_int64, c_int64, c_int, c_double, c_void_p]),
    "star_phase1_fwd": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int, POINTER(c_int64),
                                c_int, c_int, c_int, c_int64, c_int64, c_void_p, c_int, c_int64,
                                c_void_p, c_int64, c_void_p]),
    "star_phase1_fwd_check": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int, POINTER(c_int64),
                                      c_int, c_int, c_int, c_int64, c_int64, c_void_p, c_int,
                                      c_int64, c_void_p, c_void_p]),
    "star_phase1_fwd_range": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int64, c_int64,
                                      c_int, c_int, c_int, c_int64, c_int64, c_void_p, c_int,
                                      c_int64, c_void_p, c_int64, c_void_p]),
    "star_attention_dense": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int64, c_int64,
                                     c_int64, c_int, c_int, c_int, c_int, c_int64, c_int64,
                                     c_void_p, c_int64, c_void_p, c_void_p]),
    "star_kv_write": (c_int, [c_void_p, c_void_p, c_int, c_int64, c_int, c_int, c_int64, c_void_p,
                              c_void_p, c_void_p, c_int, c_int64, c_void_p]),
    "star_kv_read": (c_int, [c_void_p, c_void_p, c_int, c_void_p, c_int, c_int64, c_int64, c_int,
                             c_int, c_void_p, c_void_p, c_void_p]),
    "star_phase2_workspace_bytes": (c_int64, [c_int, c_int, c_int, c_int, c_int]),
    "star_phase2_auto_splits": (c_int, [c_int, c_int, c_int64, c_int]),
    "star_phase2_partial": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_int, c_int, c_void_p,
                                    c_void_p, c_int, c_int64, c_void_p, c_int, c_int, c_void_p,
                                    c_int64, c_int, c_void_p, c_void_p, c_int, c_void_p, c_void_p]),
    "star_merge": (c_int, [c_void_p, c_void_p, c_int, c_int64, c_int, c_void_p, c_int, c_void_p,
                           c_void_p]),
    "star_merge_strided": (c_int, [c_void_p, c_int64, c_void_p, c_int64, c_int, c_int64, c_int,
                                   c_void_p, c_int, c_void_p, c_void_p]),
    "star_exchange_box_bytes": (c_int64, [c_int, c_int64, c_int, c_int]),
    "star_ipc_get_handle": (c_int, [c_void_p, c_void_p, POINTER(c_int64)]),
    "star_ipc_open_handle": (c_int, [c_void_p, c_int64, POINTER(c_void_p)]),
    "star_ipc_close_handle": (c_int, [c_void_p, c_int64]),
    "star_phase2_partial_push": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_int, c_int,
                                         c_void_p, c_void_p, c_int, c_int64, c_void_p, c_int,
                                         c_int, c_void_p, c_int64, c_int, c_void_p, c_void_p,
                                         c_int, c_void_p, c_void_p, c_int, c_int64, c_int, c_int,
                                         c_void_p]),
    "star_phase2_exchange": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_int, c_int,
                                     c_void_p, c_void_p, c_int, c_int64, c_void_p, c_int, c_int,
                                     c_void_p, c_int64, c_int, c_void_p, c_void_p, c_int,
                                     c_void_p, c_void_p, c_int, c_int64, c_int, c_int,
                                     c_void_p]),
    "star_exchange_push": (c_int, [c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_int,
                                   c_void_p, c_int, c_int64, c_int, c_int, c_void_p]),
    "star_exchange_merge": (c_int, [c_void_p, c_int, c_int64, c_int, c_int, c_int, c_int, c_int,
                                    c_int, c_void_p, c_int, c_void_p, c_void_p]),
    "star_debug_umma_gemm": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int, c_void_p]),
}

_lib = None


def load() -> ctypes.CDLL:
    """Load libstar_attn.so (fails loudly when it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python __graft_entry__.py` (build()) "
                "or `make -C paper_2411_17116_b200/csrc`; there is no CPU fallback")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


_ERRORS = {
    STAR_ESHAPE: ShapeError,
    STAR_EDOMAIN: DomainError,
    STAR_ECONFIG: ConfigError,
    STAR_ECUDA: DeviceError,
    STAR_ENOTSUP: DeviceError,
}


def check(rc: int) -> None:
    """Map a C-ABI status onto the reference's exception classes."""
    if rc != STAR_OK:
        msg = load().star_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, DeviceError)(msg or f"star_attn status {rc}")


def call(name: str, *args) -> int:
    rc = getattr(load(), name)(*args)
    check(rc)
    return rc
