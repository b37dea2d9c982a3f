"""ctypes binding of libps_b200.so (C ABI in include/ps_b200.h).

The library is built in-tree (``__graft_entry__.build()`` or
``make -C paper_2507_23480_b200/csrc``).  There is no CPU fallback: every
entry point raises if the library or a CUDA device is missing.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PS_B200_LIB") or os.path.join(_HERE, "libps_b200.so")  # override: dev builds (TIMING=1)

PS_OK = 0
PS_ERR_INVALID = -1

_c_i64 = ctypes.c_int64
_c_i32 = ctypes.c_int32
_c_f64 = ctypes.c_double
_p = ctypes.c_void_p

# name -> (restype, argtypes); pointers are passed as integers (device addresses)
_SIGS = {
    "ps_version": (_c_i32, []),
    "ps_last_error": (ctypes.c_char_p, []),
    "ps_launch_count": (_c_i64, []),
    "ps_fps_loop": (_c_i32, [_p, _c_i64, _c_i64, _p, _p, _p, _p, _c_i64, _c_i64, _p, _c_i64, _p]),
    "ps_fps": (_c_i32, [_p, _c_i64, _c_i64, _p, _p, _p, _p, _c_i64, _c_i64, _c_i64, _p, _p]),
    "ps_set_fps_inflight": (_c_i64, [_c_i64]),
    "ps_fps_update_chunk": (_c_i32, [_p, _c_i64, _c_f64, _c_f64, _c_f64, _p, _c_i64, _c_i64, _p, _p, _p]),
    "ps_first_untaken": (_c_i32, [_p, _c_i64, _p, _p]),
    "ps_excl_workspace_bytes": (_c_i64, [_c_i64, _c_i64, _c_i64, _c_i32]),
    "ps_excl_grid_evals_offset": (_c_i64, [_c_i64, _c_i64]),
    "ps_excl_row_stride": (_c_i64, [_c_i64, _c_i64]),
    "ps_excl_build": (_c_i32, [_p, _c_i64, _c_i64, _p, _c_i32, _c_i64, _p, _p, _p, _p, _c_i64, _p, _c_i64, _p, _c_i32,
                               _p]),
    "ps_excl_build_shard": (_c_i32, [_p, _c_i64, _c_i64, _p, _c_i32, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _p, _p,
                                     _p, _p, _c_i64, _p, _p, _p]),
    "ps_early_termination_shard": (_c_i32, [_p, _p, _p, _c_i64, _p, _c_i64, _p, _p, _p, _c_i64, _p, _c_i64, _c_i64,
                                            _c_i64, _c_i64, _c_i64, _p]),
    "ps_csr_fill_workspace_bytes": (_c_i64, [_c_i64, _c_i64]),
    "ps_csr_fill": (_c_i32, [_p, _p, _p, _c_i64, _p, _c_i64, _p, _p, _p, _c_i64, _p]),
    "ps_csr_sort_rows": (_c_i32, [_p, _p, _p, _c_i64, _c_i64, _c_i64, _p, _p]),
    "ps_level_counts": (_c_i32, [_p, _p, _c_i64, _c_i64, _c_i64, _p, _c_i32, _c_i64, _p, _p]),
    "ps_thresholds": (_c_i32, [_p, _c_i64, _c_i64, _c_i64, _c_i64, _c_i32, _p, _c_i32, _p, _p, _c_i64, _p,
                               _c_i32, _p, _p, _c_i64, _p]),
    "ps_thresholds_mlp": (_c_i32, [_p, _c_i64, _c_i64, _c_i64, _c_i64, _c_i32, _p, _p, _p, _c_i32, _p, _p, _c_i64,
                                   _p]),
    "ps_sampler_workspace_bytes": (_c_i64, [_c_i64, _c_i64, _c_i32]),
    "ps_sample_predicted": (_c_i32, [_p, _p, _c_i64, _p, _c_i32, _p, _p, _c_i32, _p, _c_i64, _c_i64, _c_i64,
                                     _c_i64, _c_i64, _p, _c_i32, _p, _p, _p, _p, _p, _p]),
    "ps_earlyterm_scan": (_c_i32, [_p, _p, _p, _c_i64, _p, _c_i64, _p, _p, _c_i64, _c_i64, _c_i64, _c_i64, _p]),
    "ps_early_termination_prepare": (_c_i32, [_p, _p, _p, _c_i64, _p, _c_i64, _p, _p, _p, _c_i64, _p, _c_i64,
                                              _c_i64, _c_i64, _p]),
    "ps_ball_query_rf": (_c_i32, [_p, _p, _p, _c_i64, _p, _c_i32, _c_i32, _p, _c_i64, _c_i64, _c_i64, _c_i64,
                                  _c_i32, _p, _p, _p, _p, _p]),
    "ps_ball_query_naive": (_c_i32, [_p, _p, _c_i64, _c_i64, _c_i64, _c_i64, _c_f64, _c_i32, _p, _p, _p, _p]),
    "ps_knn_naive": (_c_i32, [_p, _p, _c_i64, _c_i64, _p, _c_i64, _c_i64, _c_i64, _c_i64, _c_i32, _p, _p, _p,
                              _p]),
    "ps_knn_rf": (_c_i32, [_p, _p, _p, _p, _c_i64, _p, _c_i64, _p, _p, _c_i64, _c_i64, _p, _c_i64, _c_i64,
                           _c_i64, _c_i64, _c_i32, _p, _p, _p, _p, _p, _p]),
    "ps_min_spacing": (_c_i32, [_p, _p, _c_i64, _c_i64, _c_i64, _c_i64, _p, _p]),
    "ps_fps_mailbox_bytes": (_c_i64, [_c_i64, _c_i32]),
    "ps_fps_split_plan": (_c_i32, [_c_i64, _c_i64, _c_i32, _c_i32, _p, _p]),
    "ps_fps_split": (_c_i32, [_p, _c_i64, _c_i64, _p, _p, _p, _p, _c_i64, _c_i64, _c_i64, _c_i32, _c_i32, _c_i32,
                              _p, ctypes.c_uint32, _c_i32, _p]),
    "ps_fps_split_loop": (_c_i32, [_p, _c_i64, _c_i64, _p, _p, _p, _p, _c_i64, _c_i64, _p, _c_i64, _c_i32, _c_i32,
                                   _c_i32, _p, ctypes.c_uint32, _c_i32, _p]),
    "ps_gather_xyz4": (_c_i32, [_p, _p, _c_i64, _c_i64, _c_i64, _c_i64, _p, _p]),
    "ps_device_alloc": (_c_i32, [_c_i64, _c_i32, _p]),
    "ps_device_free": (_c_i32, [_p]),
    "ps_ipc_handle": (_c_i32, [_p, _p]),
    "ps_ipc_open": (_c_i32, [_p, _p]),
    "ps_ipc_close": (_c_i32, [_p]),
}

EXPORTED = tuple(_SIGS)

_lock = threading.Lock()
_lib = None


class KernelError(RuntimeError):
    pass


def load(require_device: bool = False):
    """Load libps_b200.so (no device check unless ``require_device``)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"libps_b200.so not built at {LIB_PATH}; run __graft_entry__.build() "
                    "(there is no CPU fallback for the sampling path)")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    if require_device:
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("the FastPoint B200 path needs a CUDA device; none is visible")
    return _lib


def call(name: str, *args):
    """Invoke a status-returning entry point; map errors to Python exceptions."""
    lib = load(require_device=True)
    rc = getattr(lib, name)(*args)
    if rc != PS_OK:
        msg = lib.ps_last_error().decode(errors="replace")
        if rc == PS_ERR_INVALID:
            raise ValueError(f"{name}: {msg}")
        raise KernelError(f"{name}: {msg}")
    return rc


def launch_count() -> int:
    return int(load().ps_launch_count())


def raw(name: str, *args):
    return getattr(load(), name)(*args)
