"""ctypes binding of liblts_sm100.so (the C ABI in include/lts_sm100.h).

This is the only route from Python to the device: there is no CPU fallback.
If the shared library is missing or no CUDA device is visible, every call
raises.  PyTorch supplies device memory and the current stream only.
"""
from __future__ import annotations

import ctypes
import os

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LTS_SM100_LIB") or os.path.join(HERE, "liblts_sm100.so")  # override: dev variants

LTS_OK = 0
E_FIELD_NONFINITE = 1
E_BAD_DIMS = 2
E_CONSTRAINT_NOT_EXTREMUM = 3
E_LOCALIZE_NO_MIN = 4
E_VERIFY_FAILED_AT_CAP = 5
E_WORKSPACE = 6
E_CUDA = 7
E_NO_SADDLE = 8
E_INVALID = 9

MAX_REPORT_PASSES = 64
NUM_PHASES = 12
PHASES = ["order", "classify", "discover", "assemble", "localize", "integrate", "realize",
          "verify", "total", "flood_kernel"]
PH_FLOOD_LAUNCHES, PH_FLOOD_SLOTS = 10, 11  # counts reported in phase_ms slots


class lts_options_t(ctypes.Structure):
    _fields_ = [("max_iterations", ctypes.c_int32), ("restore_interior_extrema", ctypes.c_int32),
                ("collect_timing", ctypes.c_int32), ("reserved0", ctypes.c_int32),
                ("region_ni_out", ctypes.c_void_p), ("region_ni_capacity", ctypes.c_int64),
                ("reserved", ctypes.c_int32 * 4)]


class lts_pass_report_t(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("n_iter_max", ctypes.c_int32), ("seeds", ctypes.c_int64),
                ("regions", ctypes.c_int64), ("claimed", ctypes.c_int64), ("largest", ctypes.c_int64),
                ("capped", ctypes.c_int64), ("shared_saddles", ctypes.c_int64),
                ("maxima_edges", ctypes.c_int64), ("boruvka_rounds", ctypes.c_int32),
                ("big_regions", ctypes.c_int32)]


class lts_report_t(ctypes.Structure):
    _fields_ = [("ok", ctypes.c_int32), ("outer_iterations", ctypes.c_int32),
                ("restored", ctypes.c_int32), ("n_passes", ctypes.c_int32),
                ("extra_max", ctypes.c_int64), ("lost_max", ctypes.c_int64),
                ("extra_min", ctypes.c_int64), ("lost_min", ctypes.c_int64),
                ("region_ni_count", ctypes.c_int64),
                ("passes", lts_pass_report_t * MAX_REPORT_PASSES),
                ("phase_ms", ctypes.c_double * NUM_PHASES)]


class lts_regions_view_t(ctypes.Structure):
    _fields_ = [("regions", ctypes.c_int64), ("slots", ctypes.c_int64),
                ("region_ptr", ctypes.c_void_p), ("region_verts", ctypes.c_void_p),
                ("local_rank", ctypes.c_void_p), ("n_iters", ctypes.c_void_p),
                ("status", ctypes.c_void_p), ("topseed", ctypes.c_void_p)]


EXPORTS = ["lts_version", "lts_last_error", "lts_workspace_size", "lts_order_field", "lts_classify",
           "lts_remove_pass", "lts_simplify", "lts_kernel_launches", "lts_debug_big_stats", "lts_bench_kernels",
           "lts_extremum_pairs", "lts_check_field", "lts_realize_numeric", "lts_workspace_size_csr",
           "lts_classify_csr", "lts_remove_pass_csr", "lts_simplify_csr", "lts_host_scratch_size",
           "lts_simplify_host"]

_lib = None


class NativeError(RuntimeError):
    """The CUDA extension is missing or failed."""


def load():
    """Load the shared library (no GPU needed just to load it)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    P, I, I64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
    L.lts_version.restype = ctypes.c_char_p
    L.lts_last_error.restype = ctypes.c_char_p
    L.lts_kernel_launches.restype = I64
    L.lts_workspace_size.argtypes = [I, P, ctypes.POINTER(ctypes.c_size_t)]
    L.lts_order_field.argtypes = [P, I, P, P, P, P, ctypes.c_size_t, P]
    L.lts_classify.argtypes = [P, I, P, P, P, P, P]
    L.lts_remove_pass.argtypes = [I, P, P, P, I, P, ctypes.c_int32, P, P, P,
                                  ctypes.POINTER(lts_pass_report_t), ctypes.POINTER(lts_regions_view_t),
                                  P, ctypes.c_size_t, P]
    L.lts_simplify.argtypes = [P, I, P, P, I64, P, I64, P, P, P, ctypes.POINTER(lts_report_t),
                               ctypes.POINTER(lts_options_t), P, ctypes.c_size_t, P]
    L.lts_debug_big_stats.argtypes = [I, P, I]
    L.lts_bench_kernels.argtypes = [P, I, P, I, P, P, ctypes.c_size_t, P]
    L.lts_check_field.argtypes = [P, I64, P]
    L.lts_workspace_size_csr.argtypes = [I64, ctypes.POINTER(ctypes.c_size_t)]
    L.lts_classify_csr.argtypes = [P, I64, P, P, P, P, P, P, P, P, P]
    L.lts_remove_pass_csr.argtypes = [I, P, P, P, I64, P, P, ctypes.c_int32, P, P, P,
                                      ctypes.POINTER(lts_pass_report_t), ctypes.POINTER(lts_regions_view_t),
                                      P, ctypes.c_size_t, P]
    L.lts_simplify_csr.argtypes = [P, I64, P, P, P, I64, P, I64, P, P, P, ctypes.POINTER(lts_report_t),
                                   ctypes.POINTER(lts_options_t), P, ctypes.c_size_t, P]
    L.lts_realize_numeric.argtypes = [P, P, I64, ctypes.c_double, P]
    L.lts_host_scratch_size.argtypes = [I, P, I64, I64, ctypes.POINTER(ctypes.c_size_t)]
    L.lts_simplify_host.argtypes = [P, I, P, P, I64, P, I64, P, P, ctypes.POINTER(lts_report_t),
                                    ctypes.POINTER(lts_options_t), P, ctypes.c_size_t, P, ctypes.c_size_t, P]
    L.lts_extremum_pairs.argtypes = [P, P, I, P, I, ctypes.c_double, P, P, ctypes.POINTER(I64), P,
                                     ctypes.c_size_t, P]
    for name in EXPORTS:
        getattr(L, name)
    _lib = L
    return L


def last_error() -> str:
    return load().lts_last_error().decode()


def require_cuda():
    if not torch.cuda.is_available():
        raise NativeError("no CUDA device visible: the LTS path runs only on the GPU (no CPU fallback)")


def stream_ptr(device=None):
    """The current torch stream of `device` (default: the current device).
    Callers pass the device their tensors live on and run the call under
    ``torch.cuda.device(device)`` so the library works on that device."""
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def ptr(t):
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def dims_arg(dims):
    arr = (ctypes.c_int64 * 3)(*([int(d) for d in dims] + [1] * (3 - len(dims))))
    return arr


_ws_cache: dict = {}


def workspace(dims, device=None, explicit_n=None):
    """Cached device workspace for a grid shape, or for an explicit mesh of
    explicit_n vertices (caller-owned memory)."""
    dims = tuple(int(d) for d in dims) if explicit_n is None else ("csr", int(explicit_n))
    device = torch.device(device or "cuda")
    key = (dims, str(device))
    ws = _ws_cache.get(key)
    if ws is None:
        nbytes = ctypes.c_size_t(0)
        if explicit_n is None:
            check(load().lts_workspace_size(len(dims), dims_arg(dims), ctypes.byref(nbytes)))
        else:
            check(load().lts_workspace_size_csr(int(explicit_n), ctypes.byref(nbytes)))
        ws = torch.empty(int(nbytes.value), dtype=torch.uint8, device=device)
        _ws_cache.clear()  # keep one workspace alive at a time
        _ws_cache[key] = ws
    return ws


def release_workspaces():
    _ws_cache.clear()


def kernel_launches() -> int:
    return int(load().lts_kernel_launches())


def check(rc: int):
    if rc == LTS_OK:
        return
    from .errors import error_for_code
    raise error_for_code(rc, last_error())
