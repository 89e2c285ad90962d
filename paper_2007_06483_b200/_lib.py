"""ctypes binding of the sm_100a engine's C ABI (include/mtbalign_b200.h).

This is the only way the host code reaches the device: every operator in
this package calls one of these entry points with raw device pointers and
the current torch CUDA stream.  There is no CPU fallback: if the shared
library is missing or no CUDA device is present, calls raise RuntimeError.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MTB_LIB_PATH") or os.path.join(_HERE, "_lib", "libmtbalign_b200.so")

MAX_LEVELS = 16

_c_void_p = ctypes.c_void_p
_i32 = ctypes.c_int
_i64 = ctypes.c_int64
_u64p = ctypes.POINTER(ctypes.c_uint64)
_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)

# name -> argtypes (every pointer is passed as an integer address / void*).
# The status-returning functions all return int.
SIGNATURES = {
    "mtb_count_ones_packed": [_c_void_p, _i64, _i64, _c_void_p, _c_void_p],
    "mtb_count_ones_bytemap": [_c_void_p, _i64, _i64, _i64, _c_void_p, _c_void_p],
    "mtb_shifted_error_packed": [_c_void_p] * 4 + [_i64, _i64, _i64, _i64, _c_void_p, _c_void_p],
    "mtb_shifted_error_bytemap": [_c_void_p] * 4 + [_i64, _i64, _i64, _i64, _i64, _c_void_p, _c_void_p],
    "mtb_to_grayscale": [_c_void_p, _i64, _i64, _i32, _i32, _i32, _c_void_p, _i64, _i64, _c_void_p],
    "mtb_downsample_half": [_c_void_p, _i64, _i32, _i32, _c_void_p, _i64, _c_void_p],
    "mtb_histogram": [_c_void_p, _i64, _i32, _i32, _c_void_p, _c_void_p],
    "mtb_median_from_histogram": [_c_void_p, _i32, _c_void_p, _c_void_p],
    "mtb_threshold_pack": [_c_void_p, _i64, _i32, _i32, _i32, _i32, _c_void_p, _c_void_p, _c_void_p],
    "mtb_pack_mask": [_c_void_p, _i64, _i32, _i32, _c_void_p, _c_void_p],
    "mtb_unpack_bits": [_c_void_p, _i64, _i32, _i32, _c_void_p, _i64, _i32, _c_void_p],
    "mtb_shift_rgb": [_c_void_p, _i64, _i64, _i32, _i32, _i32, _c_void_p, _i32, _i32, _i32,
                      _c_void_p, _i64, _i64, _c_void_p],
    "mtb_shift_gray": [_c_void_p, _i64, _i32, _i32, _i32, _i32, _i32, _c_void_p, _i64, _c_void_p],
    "mtb_apply_lut": [_c_void_p, _c_void_p, _i64, _c_void_p, _c_void_p],
    "mtb_shifted_error_multi": [_c_void_p] * 4 + [_i64, _i64, _c_void_p, _i32, _c_void_p, _c_void_p],
    "mtb_select_candidate": [_c_void_p, _c_void_p, _i32, _i32, _i32, _c_void_p, _c_void_p],
    "mtb_pyramid_hist": [_c_void_p, _i64, _i64, _i32, _i32, _i32, _i32, _c_void_p, _c_void_p, _c_void_p],
    "mtb_threshold_levels": [_c_void_p, _c_void_p, _i32, _i32, _i32, _i32, _i32, _c_void_p, _c_void_p,
                             _c_void_p, _c_void_p, _i32, _c_void_p],
    "mtb_preprocess": [_c_void_p, _i64, _i64, _i32, _i32, _i32, _i32, _i32, _c_void_p, _c_void_p, _c_void_p,
                       _c_void_p, _c_void_p, _c_void_p, _c_void_p],
    "mtb_preprocess_maps": [_c_void_p, _i64, _i64, _i32, _i32, _i32, _i32, _i32, _c_void_p, _c_void_p,
                            _c_void_p, _c_void_p, _c_void_p],
    "mtb_find_offset_batch": [_c_void_p, _c_void_p, _i32, _i32, _c_void_p, _c_void_p, _c_void_p, _c_void_p,
                              _c_void_p],
    "mtb_search_level_rows": [_c_void_p, _i32, _i32, _i64, _i32, _i32, _i32, _i32, _i32, _c_void_p, _i64,
                              _c_void_p, _c_void_p, _i64, _c_void_p],
    "mtb_search_level_rows3": [_c_void_p, _c_void_p, _i32, _i32, _c_void_p, _c_void_p, _c_void_p, _i32, _i32, _i64,
                               _c_void_p, _c_void_p, _c_void_p, _c_void_p],
    "mtb_threshold_levels_medians": [_c_void_p, _i32, _i32, _i32, _i32, _i32, _c_void_p, _c_void_p, _c_void_p,
                                     _i32, _c_void_p],
    "mtb_decide_level": [_c_void_p, _i64, _c_void_p, _i64, _c_void_p, _c_void_p, _i64, _i32, _c_void_p],
    "mtb_align_fused": [_c_void_p, _i64, _i64, _i32, _i32, _i32, _i32, _i32, _c_void_p, _i32,
                        _c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p,
                        _c_void_p, _c_void_p],
    "mtb_align_fused_ex": [_c_void_p, _i64, _i64, _i32, _i32, _i32, _i32, _i32, _c_void_p, _i32,
                           _c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p,
                           _c_void_p, _c_void_p, _c_void_p],
    "mtb_stream_write_u32": [_c_void_p, ctypes.c_uint32, _c_void_p],
}

# Non-status entry points.
AUX_SIGNATURES = {
    "mtb_last_error": ([], ctypes.c_char_p),
    "mtb_abi_version": ([], ctypes.c_int),
    "mtb_launch_count": ([], ctypes.c_uint64),
    "mtb_plan_levels": ([_i32, _i32, _i32, _i64p, _i64p], ctypes.c_int),
    "mtb_align_fused_workspace": ([_i32, _i32, _i32, _i64p, _i64p], ctypes.c_int),
    "mtb_align_fused_sync_words": ([_i32, _i32, _i32], ctypes.c_int64),
    "mtb_align_fused_images_per_launch": ([_i32, _i32], ctypes.c_int),
    "mtb_align_fused_launches": ([_i32, _i32, _i32, _i32, _c_void_p, _i32], ctypes.c_int),
    "mtb_preprocess_maps_cluster": ([_i32, _i32, _i32], ctypes.c_int),
    "mtb_preprocess_maps_shape": ([_i32, _i32, _i32, _c_void_p], ctypes.c_int),
}

_lock = threading.Lock()
_lib = None


class EngineError(RuntimeError):
    """A CUDA-side failure reported through the C ABI."""


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load (once) and type the shared library; raises RuntimeError if absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise RuntimeError(
                f"CUDA engine library not built: {path} is missing; run "
                "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
        lib = ctypes.CDLL(path)
        # an experiment build (MTB_LIB_PATH, tools/ab.sh) may predate newer entry points
        lenient = bool(os.environ.get("MTB_LIB_PATH"))
        sigs = [(n, a, ctypes.c_int) for n, a in SIGNATURES.items()] + \
               [(n, a, r) for n, (a, r) in AUX_SIGNATURES.items()]
        for name, argtypes, restype in sigs:
            if lenient and not hasattr(lib, name):
                continue
            fn = getattr(lib, name)
            fn.argtypes = argtypes
            fn.restype = restype
        _lib = lib
        return lib


def exported_symbols() -> list[str]:
    return sorted(list(SIGNATURES) + list(AUX_SIGNATURES))


def call(name: str, *args) -> None:
    """Invoke a status-returning entry point; raise on failure.

    MTB_EINVAL maps to ValueError (argument errors, as the reference's own
    validation raises), MTB_ECUDA to EngineError.
    """
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        msg = lib.mtb_last_error().decode(errors="replace")
        if rc == 1:
            raise ValueError(f"{name}: {msg}")
        raise EngineError(f"{name} failed ({rc}): {msg}")


def launch_count() -> int:
    return int(load().mtb_launch_count())


def plan_levels(width: int, height: int, requested: int):
    """Level count and arena geometry (mtb_plan_levels); None if invalid."""
    lib = load()
    geom = np.zeros((MAX_LEVELS, 6), dtype=np.int64)
    sizes = np.zeros(3, dtype=np.int64)
    n = lib.mtb_plan_levels(int(width), int(height), int(requested),
                            geom.ctypes.data_as(_i64p), sizes.ctypes.data_as(_i64p))
    if n < 1:
        return None
    return n, geom[:n].copy(), sizes.copy()


def require_cuda():
    """Import torch and check a CUDA device exists (no CPU fallback)."""
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("mtbalign-b200 requires a CUDA device (sm_100a); none is available")
    load()
    return torch


def stream_handle(torch_mod=None) -> int:
    import torch

    return torch.cuda.current_stream().cuda_stream
