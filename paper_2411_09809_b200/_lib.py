"""ctypes binding of the sm_100a C-ABI library (include/glare_b200.h).

The library is built in-tree (``make`` or ``__graft_entry__.build()``) into
``paper_2411_09809_b200/_lib/libglare_b200.so``.  There is no fallback: if the
library or a CUDA device is missing, ``lib()`` raises ``RuntimeError``.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# GLARE_B200_LIB points at an alternative build (tuning sweeps in tools/).
LIB_PATH = os.environ.get("GLARE_B200_LIB") or os.path.join(_HERE, "_lib", "libglare_b200.so")

GLR_OK = 0
GLR_EARG = 1
GLR_ECUDA = 2
GLR_ENCCL = 3
GLR_EINVARIANT = 4
GLR_EFALLBACK = 8
GLR_EPARSE = 16

# (name, restype, argtypes) for every symbol include/glare_b200.h declares.
_c = ctypes
SIGNATURES = {
    "glr_version": (_c.c_int, []),
    "glr_last_error": (_c.c_char_p, []),
    "glr_occlusion_tile": (_c.c_int, []),
    "glr_occlusion_units": (_c.c_uint64, [_c.c_int64]),
    "glr_occlusion_count": (
        _c.c_int,
        [_c.c_void_p, _c.c_int64, _c.c_double, _c.c_uint64, _c.c_uint64, _c.c_void_p, _c.c_void_p],
    ),
    "glr_crossing_tile": (_c.c_int, []),
    "glr_crossing_band": (_c.c_int, []),
    "glr_crossing_chunk": (_c.c_uint64, [_c.c_uint64, _c.c_int]),
    "glr_allreduce_sum_f64": (
        _c.c_int, [_c.c_int, _c.POINTER(_c.c_int), _c.POINTER(_c.c_void_p), _c.c_int]),
    "glr_nccl_id_bytes": (_c.c_int, []),
    "glr_nccl_unique_id": (_c.c_int, [_c.c_void_p]),
    "glr_nccl_comm_init": (_c.c_int, [_c.c_void_p, _c.c_int, _c.c_int, _c.POINTER(_c.c_void_p)]),
    "glr_allreduce_sum_f64_comm": (_c.c_int, [_c.c_void_p, _c.c_void_p, _c.c_int, _c.c_void_p]),
    "glr_nccl_comm_destroy": (_c.c_int, [_c.c_void_p]),
    "glr_crossing_units": (_c.c_uint64, [_c.c_int64]),
    "glr_crossing_records_bytes": (_c.c_size_t, [_c.c_int64, _c.c_int64]),
    "glr_crossing_prepare": (
        _c.c_int,
        [_c.c_void_p, _c.c_int64, _c.c_void_p, _c.c_int64, _c.c_void_p, _c.c_void_p],
    ),
    "glr_crossing_pairs": (
        _c.c_int,
        [_c.c_void_p, _c.c_int64, _c.c_int64, _c.c_int, _c.c_double, _c.c_uint64,
         _c.c_uint64, _c.c_void_p, _c.c_void_p],
    ),
    "glr_crossing_scan": (
        _c.c_int,
        [_c.c_void_p, _c.c_int64, _c.c_void_p, _c.c_int64, _c.c_int, _c.c_double,
         _c.c_uint64, _c.c_uint64, _c.c_void_p, _c.c_void_p],
    ),
    "glr_edge_length_variation": (
        _c.c_int,
        [_c.c_void_p, _c.c_int64, _c.c_void_p, _c.c_int64, _c.c_void_p, _c.c_void_p],
    ),
    "glr_minimum_angle": (
        _c.c_int,
        [_c.c_void_p, _c.c_int64, _c.c_void_p, _c.c_int64, _c.c_void_p, _c.c_void_p],
    ),
    "glr_crossing_fast_path": (_c.c_int, [_c.c_void_p, _c.c_void_p]),
    "glr_crossing_set_mode": (_c.c_int, [_c.c_void_p, _c.c_int, _c.c_void_p]),
    "glr_occlusion_set_filter": (_c.c_int, [_c.c_int]),
    "glr_parse_edgelist": (_c.c_int, [_c.c_char_p, _c.c_size_t, _c.c_void_p, _c.c_int64,
                                      _c.POINTER(_c.c_int64)]),
    "glr_parse_layout": (_c.c_int, [_c.c_char_p, _c.c_size_t, _c.c_void_p, _c.c_void_p,
                                    _c.c_int64, _c.POINTER(_c.c_int64)]),
    "glr_parse_status": (_c.c_int, [_c.c_void_p]),
    "glr_strip_crossings": (_c.c_int, [_c.c_void_p, _c.c_int64, _c.c_void_p, _c.c_int64,
                                       _c.c_void_p, _c.c_int64, _c.c_int, _c.c_int,
                                       _c.c_double, _c.c_void_p, _c.c_void_p]),
    "glr_selftest_division": (_c.c_int, [_c.c_uint64, _c.c_uint64,
                                         _c.POINTER(_c.c_uint64), _c.c_void_p]),
    "glr_fr_layout": (_c.c_int, [_c.c_void_p, _c.c_int64, _c.c_void_p, _c.c_void_p,
                                 _c.c_int64, _c.c_int, _c.c_double, _c.c_void_p]),
    "glr_take_launch_count": (_c.c_uint64, []),
    "glr_crossing_pairs_interleaved": (
        _c.c_int,
        [_c.c_void_p, _c.c_int64, _c.c_int64, _c.c_int, _c.c_double, _c.c_void_p, _c.c_uint64,
         _c.c_int, _c.c_int, _c.c_void_p, _c.c_void_p],
    ),
    "glr_crossing_tile_weights": (
        _c.c_int, [_c.c_void_p, _c.c_int64, _c.c_int64, _c.c_double, _c.c_void_p, _c.c_void_p]),
    "glr_spatial_sort_edges": (
        _c.c_int,
        [_c.c_void_p, _c.c_int64, _c.c_void_p, _c.c_int64, _c.c_void_p, _c.c_void_p],
    ),
    "glr_theta_sort_edges": (
        _c.c_int,
        [_c.c_void_p, _c.c_int64, _c.c_void_p, _c.c_int64, _c.c_int64, _c.c_void_p,
         _c.c_void_p],
    ),
    "glr_spatial_set_kd": (_c.c_int, [_c.c_int]),
    "glr_crossing_sub_mask_bytes": (_c.c_int, []),
    "glr_crossing_sub_quarters": (_c.c_int, []),
    "glr_spatial_sort_vertices": (
        _c.c_int, [_c.c_void_p, _c.c_int64, _c.c_void_p, _c.c_void_p]),
    "glr_crossing_candidates": (
        _c.c_int,
        [_c.c_void_p, _c.c_int64, _c.c_int64, _c.c_void_p, _c.c_uint64,
         _c.POINTER(_c.c_uint64), _c.c_void_p],
    ),
    "glr_crossing_pairs_list": (
        _c.c_int,
        [_c.c_void_p, _c.c_int64, _c.c_int64, _c.c_int, _c.c_double, _c.c_void_p,
         _c.c_uint64, _c.c_uint64, _c.c_uint64, _c.c_void_p, _c.c_void_p],
    ),
    "glr_crossing_candidates_classified": (
        _c.c_int,
        [_c.c_void_p, _c.c_int64, _c.c_int64, _c.c_void_p, _c.c_void_p, _c.c_uint64,
         _c.POINTER(_c.c_uint64), _c.c_void_p],
    ),
    "glr_crossing_candidates_rows": (
        _c.c_int,
        [_c.c_void_p, _c.c_int64, _c.c_int64, _c.c_void_p, _c.c_void_p, _c.c_uint64,
         _c.POINTER(_c.c_uint64), _c.c_int, _c.c_int, _c.c_void_p],
    ),
    "glr_crossing_pairs_classified": (
        _c.c_int,
        [_c.c_void_p, _c.c_int64, _c.c_int64, _c.c_int, _c.c_double, _c.c_void_p, _c.c_void_p,
         _c.c_uint64, _c.c_uint64, _c.c_uint64, _c.c_uint64, _c.c_int, _c.c_int, _c.c_void_p,
         _c.c_void_p],
    ),
    "glr_occlusion_candidates": (
        _c.c_int,
        [_c.c_void_p, _c.c_int64, _c.c_double, _c.c_void_p, _c.c_uint64,
         _c.POINTER(_c.c_uint64), _c.c_void_p],
    ),
    "glr_occlusion_count_list": (
        _c.c_int,
        [_c.c_void_p, _c.c_int64, _c.c_double, _c.c_void_p, _c.c_uint64, _c.c_uint64,
         _c.c_uint64, _c.c_void_p, _c.c_void_p],
    ),
}

_lock = threading.Lock()
_handle = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """dlopen the library and declare every exported signature.  Does not
    touch the GPU, so it works on a CPU-only host (ABI tests)."""
    if not os.path.exists(path):
        raise RuntimeError(
            f"glare_b200 CUDA library not built: {path} is missing "
            "(run `make` or __graft_entry__.build())"
        )
    h = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(h, name)
        fn.restype = res
        fn.argtypes = args
    return h


_host_handle = None


def host_lib() -> ctypes.CDLL:
    """The library for its host-only entry points (the native loaders): no
    CUDA device needed."""
    global _host_handle
    if _host_handle is None:
        with _lock:
            if _host_handle is None:
                _host_handle = load_library(os.environ.get("GLARE_B200_LIB") or LIB_PATH)
    return _host_handle


def lib() -> ctypes.CDLL:
    """The loaded library, after checking that a CUDA device is usable."""
    global _handle
    if _handle is None:
        with _lock:
            if _handle is None:
                import torch

                if not torch.cuda.is_available():
                    raise RuntimeError(
                        "glare_b200 needs a CUDA device (B200, sm_100a); none is visible"
                    )
                _handle = load_library()
    return _handle


def check(rc: int, what: str) -> None:
    """Map a C-ABI status code to the reference's exception classes."""
    if rc == GLR_OK:
        return
    from .model import InvariantError, ParameterError

    msg = host_lib().glr_last_error()
    msg = msg.decode() if msg else ""
    if rc == GLR_EARG:
        raise ParameterError(f"{what}: {msg}")
    if rc == GLR_EINVARIANT:
        raise InvariantError(f"{what}: {msg}")
    raise RuntimeError(f"{what} failed (code {rc}): {msg}")
