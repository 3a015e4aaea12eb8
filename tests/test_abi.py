"""C ABI: the library loads, exports every declared symbol, validates on the host."""
import ctypes
import glob
import os
import re

import pytest

from paper_2507_19926_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(h).read()
        names |= set(re.findall(r"\b(tm_[a-z0-9_]+)\s*\(", text))
    return names


def test_library_exports_header_symbols():
    lib = _lib.load()
    declared = _declared()
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(lib, name), name
    assert set(_lib.EXPORTED) == declared


def test_version_and_kernel_names():
    lib = _lib.load()
    assert b"sm_100a" in lib.tm_version()
    assert lib.tm_kernel_name(1) == b"oblivious"
    assert lib.tm_kernel_name(3) == b"select"


def test_dispatch_query_routes():
    lib = _lib.load()
    assert lib.tm_dispatch_query(8, 5, 5, 0) == 1          # auto, small k -> oblivious kernel
    assert lib.tm_dispatch_query(8, 3, 3, 0) == 6          # k = 3 -> specialised network
    assert lib.tm_dispatch_query(16, 9, 9, 3) == 3         # oracle -> brute-force select
    assert lib.tm_dispatch_query(8, 3, 5, 1) in (1, 2, 3)  # rectangular
    assert lib.tm_dispatch_query(12, 3, 3, 0) == 0         # bad width
    assert lib.tm_dispatch_query(8, 4, 4, 0) == 0          # even kernel


def test_dispatch_table_crossovers():
    """auto: oblivious below the measured crossover, data-aware from it on."""
    lib = _lib.load()
    name = lambda b, k, v=0: lib.tm_kernel_name(lib.tm_dispatch_query(b, k, k, v)).decode()
    assert [name(8, k) for k in (11, 13, 75)] == ["oblivious", "histogram", "histogram"]
    assert [name(16, k) for k in (25, 27, 75)] == ["oblivious", "rank", "rank"]
    assert [name(32, k) for k in (21, 23, 75)] == ["oblivious", "rank", "rank"]
    assert name(8, 9, 2) == "histogram" and name(16, 9, 2) == "rank"   # variant "aware"
    assert name(8, 17, 1) == "oblivious"                               # variant "oblivious"
    assert name(32, 5, 3) == "select"                                  # variant "oracle"


def test_oblivious_variant_above_27_is_reported_as_select():
    """variant "oblivious" runs a comparator-network kernel for k <= 27; above,
    the exact per-pixel radix selection (the same results) -- and says so."""
    lib = _lib.load()
    name = lambda b, k: lib.tm_kernel_name(lib.tm_dispatch_query(b, k, k, 1)).decode()
    from paper_2507_19926_b200 import dispatch_query
    import numpy as np
    for bits, dt in ((8, np.uint8), (16, np.uint16), (32, np.uint32)):
        assert name(bits, 27) == "oblivious"
        assert [name(bits, k) for k in (29, 49, 75)] == ["select"] * 3
        assert dispatch_query(dt, 29, "oblivious") == "select"


def test_host_validation_without_gpu():
    """Argument errors are reported before any CUDA call (no GPU needed)."""
    lib = _lib.load()
    buf = ctypes.create_string_buffer(64)
    p = ctypes.addressof(buf)
    assert lib.tm_median2d(p, 8, p, 8, 8, 8, 12, 3, 0, None) == _lib.TM_ETYPE
    assert lib.tm_median2d(p, 8, p, 8, 8, 8, 8, 4, 0, None) == _lib.TM_EINVAL
    assert b"odd" in lib.tm_last_error()
    assert lib.tm_median2d(p, 8, p, 8, 0, 8, 8, 3, 0, None) == _lib.TM_EINVAL
    assert lib.tm_median2d(p, 4, p, 8, 8, 8, 8, 3, 0, None) == _lib.TM_EINVAL  # pitch < row
    assert lib.tm_median2d(p, 8, p, 8, 8, 8, 8, 3, 9, None) == _lib.TM_EINVAL  # variant
    assert lib.tm_median2d_band(p, 8, 8, 4, 8, p, 8, 8, 1, 8, 3, 3, 0, None) == _lib.TM_EINVAL
    with pytest.raises(ValueError):
        _lib.check(_lib.TM_EINVAL)
    with pytest.raises(TypeError):
        _lib.check(_lib.TM_ETYPE)
    with pytest.raises(RuntimeError):
        _lib.check(_lib.TM_ECUDA)
