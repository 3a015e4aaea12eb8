"""ctypes binding of the C ABI (include/tilemedian_b200.h).

The shared library is built in-tree (``python -m paper_2507_19926_b200.build``
or ``__graft_entry__.build()``).  There is no CPU fallback: if the library is
missing or CUDA is unusable every entry point raises.
"""
from __future__ import annotations

import ctypes
import os
import threading

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TMB_LIB", os.path.join(_PKG, "libtilemedian_b200.so"))

VARIANT_CODES = {"auto": 0, "oblivious": 1, "aware": 2, "oracle": 3}
KERNEL_NAMES = {0: "none", 1: "oblivious", 2: "multipass", 3: "select", 4: "histogram", 5: "rank", 6: "med3"}
KERNEL_CODES = {v: k for k, v in KERNEL_NAMES.items()}
TM_OK, TM_EINVAL, TM_ETYPE, TM_ECUDA = 0, 1, 2, 3

_lock = threading.Lock()
_lib = None

c_i32, c_i64, c_vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p

_SIGS = {
    "tm_median2d": (ctypes.c_int, [c_vp, c_i64, c_vp, c_i64, c_i32, c_i32, c_i32, c_i32, c_i32, c_vp]),
    "tm_median2d_rect": (ctypes.c_int, [c_vp, c_i64, c_vp, c_i64, c_i32, c_i32, c_i32, c_i32, c_i32,
                                        c_i32, c_vp]),
    "tm_median2d_planes": (ctypes.c_int, [c_vp, c_i64, c_vp, c_i64, c_i32, c_i32, c_i32, c_i32,
                                          c_i32, c_i32, c_vp]),
    "tm_median2d_band": (ctypes.c_int, [c_vp, c_i64, c_i32, c_i32, c_i32, c_vp, c_i64, c_i32, c_i32,
                                        c_i32, c_i32, c_i32, c_i32, c_vp]),
    "tm_median2d_host": (ctypes.c_int, [c_vp, c_i64, c_vp, c_i64, c_i32, c_i32, c_i32, c_i32, c_i32,
                                        c_i32, c_i32, c_i32]),
    "tm_median2d_host_budget": (ctypes.c_int, [c_vp, c_i64, c_vp, c_i64, c_i32, c_i32, c_i32, c_i32,
                                               c_i32, c_i32, c_i32, c_i32, c_i64]),
    "tm_median2d_host_multi": (ctypes.c_int, [c_vp, c_i64, c_vp, c_i64, c_i32, c_i32, c_i32, c_i32,
                                              c_i32, c_i32, c_i32, c_vp, c_i32]),
    "tm_median2d_host_frames": (ctypes.c_int, [c_vp, c_i64, c_i64, c_vp, c_i64, c_i64, c_i32, c_i32,
                                               c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_vp,
                                               c_i32]),
    "tm_median2d_bands": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_i32, c_i32,
                                         c_i32, c_i32, c_i32, c_i32, c_vp]),
    "tm_host_alloc": (c_vp, [c_i64]),
    "tm_host_free": (ctypes.c_int, [c_vp]),
    "tm_dispatch_query": (ctypes.c_int, [c_i32, c_i32, c_i32, c_i32]),
    "tm_kernel_name": (ctypes.c_char_p, [c_i32]),
    "tm_force_kernel": (ctypes.c_int, [c_i32]),
    "tm_launch_count": (ctypes.c_int64, []),
    "tm_last_error": (ctypes.c_char_p, []),
    "tm_version": (ctypes.c_char_p, []),
}

EXPORTED = tuple(_SIGS)


def load():
    """Load the extension; raises RuntimeError when it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"CUDA extension not built ({LIB_PATH} missing); run "
                    "`python -m paper_2507_19926_b200.build` -- there is no CPU fallback")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def check(rc: int) -> None:
    """Translate a C ABI status into the reference's Python exceptions."""
    if rc == TM_OK:
        return
    msg = load().tm_last_error().decode(errors="replace")
    if rc == TM_EINVAL:
        raise ValueError(msg)
    if rc == TM_ETYPE:
        raise TypeError(msg)
    raise RuntimeError(msg)
