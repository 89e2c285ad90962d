"""The C-ABI boundary on CPU: the library loads, exports every symbol the
header declares, plans pyramids exactly like the reference, and rejects bad
arguments before touching the device.  No kernel launches."""

import ctypes
import os
import re

import numpy as np
import pytest

import mtb_oracle as orc
from paper_2007_06483_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "mtbalign_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mtb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_lib.exported_symbols())


def test_abi_version():
    assert _lib.load().mtb_abi_version() == 1


@pytest.mark.parametrize("w,h,L", [(1024, 768, 6), (6000, 4000, 6), (4000, 3000, 6), (2560, 1440, 6), (64, 64, 6),
                                   (16, 16, 3), (17, 33, 10), (40000, 25000, 10), (129, 4097, 16), (1023, 769, 5)])
def test_plan_matches_reference_pyramid(w, h, L):
    n, geom, sizes = _lib.plan_levels(w, h, L)
    assert n == min(L, orc.max_levels(w, h))
    gw, gh = w, h
    prev_gray_end, prev_bit_end = 0, 0
    for k in range(n):
        lw, lh, pitch, goff, nw64, boff = (int(v) for v in geom[k])
        assert (lw, lh) == (gw, gh)                  # floor halving, pyramid.py:29
        assert pitch % 128 == 0 and pitch >= lw
        assert nw64 == (lw + 63) // 64                # bitmap.py:35
        assert goff % 256 == 0 and goff >= prev_gray_end
        assert boff % 32 == 0 and boff >= prev_bit_end
        prev_gray_end, prev_bit_end = goff + pitch * lh, boff + nw64 * lh
        gw, gh = gw // 2, gh // 2
    assert sizes[0] >= prev_gray_end and sizes[1] >= prev_bit_end


def test_plan_rejects_small_or_zero_levels():
    assert _lib.plan_levels(15, 100, 6) is None      # pyramid.py:55-56
    assert _lib.plan_levels(100, 15, 6) is None
    assert _lib.plan_levels(100, 100, 0) is None     # pyramid.py:52-53


def test_invalid_arguments_fail_before_the_device():
    lib = _lib.load()
    rc = lib.mtb_preprocess(None, 0, 0, 64, 64, 1, 6, 4, None, None, None, None, None, None, None)
    assert rc == 1 and b"null" in lib.mtb_last_error()
    with pytest.raises(ValueError):
        _lib.call("mtb_find_offset_batch", None, None, 0, 1, None, None, None, None, None)
    with pytest.raises(ValueError):
        _lib.call("mtb_downsample_half", 1, 1, 1, 1, 1, 1, None)   # 1x1 cannot be halved
    rc = lib.mtb_pyramid_hist(ctypes.c_void_p(16), 3 * 8, 0, 8, 8, 1, 6, ctypes.c_void_p(16), ctypes.c_void_p(16),
                              None)
    assert rc == 1 and b"16x16" in lib.mtb_last_error()


def test_error_message_is_thread_local():
    import threading

    lib = _lib.load()
    lib.mtb_preprocess(None, 0, 0, 64, 64, 1, 6, 4, None, None, None, None, None, None, None)
    seen = []
    t = threading.Thread(target=lambda: seen.append(lib.mtb_last_error()))
    t.start()
    t.join()
    assert seen == [b""]
    assert lib.mtb_last_error() != b""


def test_missing_library_fails_loudly(tmp_path):
    import importlib

    mod = importlib.import_module("paper_2007_06483_b200._lib")
    with pytest.raises(RuntimeError, match="not built"):
        saved = mod._lib
        mod._lib = None
        try:
            mod.load(str(tmp_path / "absent.so"))
        finally:
            mod._lib = saved
