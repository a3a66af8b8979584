"""ctypes binding of ``_lib/libtwgemm.so`` (C ABI in include/tw_gemm.h).

This is the only place the package touches the native library.  There is no
CPU fallback: if the library or a CUDA device is missing, every entry point
raises :class:`DeviceError`.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

from .errors import DeviceError, raise_for_status

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libtwgemm.so"

TW_F32, TW_F16, TW_BF16 = 0, 1, 2
TW_LAYOUT_NATURAL, TW_LAYOUT_PLAN = 0, 1
SCHEDULES = {"lpt": 0, "round_robin": 1}

_c_int = ctypes.c_int
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_vp = ctypes.c_void_p
_u32p = ctypes.POINTER(ctypes.c_uint32)
_i32p = ctypes.POINTER(ctypes.c_int32)
_i64p = ctypes.POINTER(ctypes.c_int64)
_f32p = ctypes.POINTER(ctypes.c_float)


class PlanInfo(ctypes.Structure):
    _fields_ = [("k", _i32), ("n", _i32), ("g", _i32), ("n_tiles", _i32), ("n_sub", _i32),
                ("bn", _i32), ("kp", _i32), ("n_condensed", _i32), ("n_union", _i32),
                ("compute_dtype", _i32), ("nnz", _i64), ("kept_macs_per_token", _i64),
                ("sm_count", _i32), ("has_overlay", _i32), ("row_runs", _i32),
                ("row_copies", _i32), ("sm_budget", _i32), ("stage_work", _i64),
                ("sparse_payload", _i32), ("splitk_max", _i32),
                ("splitk_max_tokens", _i32), ("splitk_min_steps", _i32)]


# name -> (restype, argtypes); must match include/tw_gemm.h exactly
SIGNATURES = {
    "tw_plan_create_cto": (_c_int, [ctypes.POINTER(_vp), _i32, _i32, _i32, _i32, _u32p, _u32p,
                                    _u32p, _i32, _u32p, _i32, _f32p, _i32, _i32, _i32, _vp]),
    "tw_plan_create_cto_ex": (_c_int, [ctypes.POINTER(_vp), _i32, _i32, _i32, _i32, _u32p, _u32p,
                                       _u32p, _i32, _u32p, _i32, _f32p, _i32, _i32, _i32, _i32p,
                                       _i32, _i32p, _vp]),
    "tw_plan_output_groups": (_c_int, [_vp, _i32p]),
    "tw_plan_save": (_c_int, [_vp, _vp, ctypes.POINTER(ctypes.c_uint64)]),
    "tw_plan_load": (_c_int, [ctypes.POINTER(_vp), _vp, ctypes.c_uint64, _vp]),
    "tw_plan_attach_overlay": (_c_int, [_vp, _i32, _i32, _i64, _i64p, _i64p, _f32p, _vp]),
    "tw_plan_get_info": (_c_int, [_vp, ctypes.POINTER(PlanInfo)]),
    "tw_plan_set_sm_budget": (_c_int, [_vp, _i32]),
    "tw_plan_estimate": (_c_int, [_vp, _i32, _i64, _i64p, _i32p]),
    "tw_plan_condensed_columns": (_c_int, [_vp, _i32p]),
    "tw_plan_union_columns": (_c_int, [_vp, _i32p]),
    "tw_gemm": (_c_int, [_vp, _vp, _i64, _i64, _vp, _i64, _i32, _vp]),
    "tw_gemm_ex": (_c_int, [_vp, _vp, _i64, _i64, _vp, _i64, _i32, _i32, _vp]),
    "tw_gemm_group": (_c_int, [ctypes.POINTER(_vp), _i32, ctypes.POINTER(_vp), _i64p, _i32p,
                               ctypes.POINTER(_vp), _i64p, _i64, _i32, _vp]),
    "tw_gemm_tew_group": (_c_int, [ctypes.POINTER(_vp), _i32, ctypes.POINTER(_vp), _i64p, _i32p,
                                   ctypes.POINTER(_vp), _i64p, ctypes.POINTER(_vp),
                                   ctypes.POINTER(ctypes.c_uint64), _i64, _i32, _vp]),
    "tw_plan_prepare": (_c_int, [_vp, _vp, _i32, _i64, _i64, _vp, _i64, _vp]),
    "tw_plan_row_order": (_c_int, [_vp, _i32p]),
    "tw_plan_permute_rows": (_c_int, [_vp, _vp, _i64, _i64, _vp, _i64, _vp]),
    "tw_gemm_tew": (_c_int, [_vp, _vp, _i64, _i64, _vp, _i64, _i32, _vp]),
    "tw_gemm_tew_ws": (_c_int, [_vp, _vp, _i64, _i64, _vp, _i64, _i32, _vp, ctypes.c_uint64, _vp]),
    "tw_gemm_tew_ex": (_c_int, [_vp, _vp, _i64, _i64, _vp, _i64, _i32, _vp, ctypes.c_uint64, _i32,
                                _vp]),
    "tw_gemm_tew_reuse": (_c_int, [_vp, _vp, _i64, _i64, _vp, _i64, _i32p, _vp, _i64, _i32, _i32,
                                   _vp]),
    "tw_plan_tew_workspace_bytes": (_c_int, [_vp, _i64, _i32, ctypes.POINTER(ctypes.c_uint64)]),
    "tw_transpose_cast": (_c_int, [_vp, _i32, _i64, _i64, _i64, _vp, _i32, _i64, _vp]),
    "tw_plan_destroy": (None, [_vp]),
    "tw_debug_set_trace": (None, [_vp]),
    "tw_last_error": (ctypes.c_char_p, []),
    "tw_abi_version": (_i32, []),
}

_lock = threading.Lock()
_lib = None


def load_library(path: Path = LIB_PATH) -> ctypes.CDLL:
    """Load (once) and type the C ABI.  Does not touch the GPU.
    ``TW_LIB_PATH`` (diagnostics: A/B builds of the same ABI) overrides the path."""
    global _lib
    path = Path(os.environ.get("TW_LIB_PATH", str(path)))
    with _lock:
        if _lib is not None:
            return _lib
        if not path.exists():
            raise DeviceError(
                f"{path} is missing: build it with `python __graft_entry__.py` "
                "(or paper_2402_10876_b200._build.build_native())")
        lib = ctypes.CDLL(str(path))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(status: int) -> None:
    """Raise the mapped exception for a non-zero status."""
    if status:
        msg = load_library().tw_last_error()
        raise_for_status(status, msg.decode() if msg else "")


_torch_ok = None


def require_cuda():
    """Return torch with a usable CUDA device, or raise DeviceError (the
    device check runs once per process)."""
    global _torch_ok
    if _torch_ok is not None:
        return _torch_ok
    import torch

    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the TW/TEW matmul runs only on the GPU "
                          "(there is deliberately no CPU fallback)")
    _torch_ok = torch
    return torch


def stream_handle(stream=None) -> int:
    torch = require_cuda()
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(arr, ctype):
    """ctypes pointer to a contiguous numpy array's data."""
    return arr.ctypes.data_as(ctypes.POINTER(ctype))
