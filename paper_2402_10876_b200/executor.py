"""The "matmul" step on B200: the reference executor API backed by sm_100a kernels.

Keeps the call signatures of reference executor.py so it drops in for the
TW/TEW path:

* :func:`gemm_tile_sparse` -- executor.py:135-146
* :func:`gemm_cto`         -- executor.py:149-177
* :func:`execute_batched`  -- executor.py:230-265 (+ :func:`schedule_tiles` 206-227)
* :func:`gemm_tew`         -- executor.py:180-203
* :class:`GemmOutput`      -- executor.py:68-80
* :class:`ExecutionTrace`  -- executor.py:83-118
* :func:`relative_error`   -- executor.py:278-288

Every product runs in ``libtwgemm.so`` (K1 ``tw_gather_gemm`` for TW, K1 +
K2 ``tw_residual`` for TEW) on the current CUDA device and stream.  Numerics
contract: operands are rounded once to ``compute_dtype``
(fp16 default, bf16 optional), products accumulate in fp32 in TMEM, and the
output is fp32 unless ``out_dtype`` asks for fp16/bf16.  The three TW entry
points launch the same deterministic kernel, so -- as in the reference --
their outputs are bit-identical to each other.

Outputs live on the GPU: ``GemmOutput.condensed`` is an M x N' torch view of
the kernel's native C'^T (N' x M) buffer.
"""

from __future__ import annotations

import weakref
from dataclasses import dataclass
from typing import List, Optional, Tuple, Union

import numpy as np

from . import _native
from .core import ACC_DTYPE, IndexMask, as_matrix
from .errors import DeviceError, InvalidInputError
from .formats import CtoEncoding, encode_cto
from .patterns import SparseOverlay, TileSparseMatrix

_DTYPE_CODES = {"fp32": _native.TW_F32, "fp16": _native.TW_F16, "bf16": _native.TW_BF16}


def _torch():
    return _native.require_cuda()


def _torch_dtype(name: str):
    torch = _torch()
    return {"fp32": torch.float32, "fp16": torch.float16, "bf16": torch.bfloat16}[name]


def _dtype_name(dt) -> str:
    """Accept 'fp16' / torch.float16 / np.float16 style names."""
    if isinstance(dt, str):
        if dt in _DTYPE_CODES:
            return dt
        raise InvalidInputError(f"unknown dtype {dt!r}")
    torch = _torch()
    table = {torch.float32: "fp32", torch.float16: "fp16", torch.bfloat16: "bf16"}
    if dt in table:
        return table[dt]
    raise InvalidInputError(f"unsupported dtype {dt!r}")


# ----------------------------------------------------------------------------
# device plan (GPU weight format)
# ----------------------------------------------------------------------------

class TwPlan:
    """Device-resident TW weight (plus optional TEW overlay).

    Built from a :class:`CtoEncoding` (the reference's compressed format,
    formats.py:82-181); the C library validates it exactly like
    ``gemm_cto`` does and derives the GPU layout: per-tile int32 gather lists
    padded to a multiple of 64 and the K-major fp16/bf16 payload.
    """

    def __init__(self, enc: CtoEncoding, overlay: Optional[SparseOverlay] = None,
                 compute_dtype: str = "fp16", schedule: str = "lpt",
                 row_layout: str = "natural", row_groups=None, out_order=None):
        torch = _torch()
        lib = _native.load_library()
        if schedule not in _native.SCHEDULES:
            raise InvalidInputError(f"unknown strategy {schedule!r}")
        if row_layout not in ("natural", "runs"):
            raise InvalidInputError(f"row_layout must be 'natural' or 'runs', got {row_layout!r}")
        self.row_layout = row_layout
        self.compute_dtype = _dtype_name(compute_dtype)
        # fp32: the operands are split into fp16 hi + lo pairs (three fp16
        # products, fp32-class accuracy); the kernels read fp16
        self.split = self.compute_dtype == "fp32"
        self.operand_dtype = "fp16" if self.split else self.compute_dtype
        self.schedule = schedule
        self.device = torch.cuda.current_device()
        self.original_dims = enc.original_dims
        k, n = enc.original_dims
        rc = np.ascontiguousarray(enc.row_counts, dtype=np.uint32)
        cc = np.ascontiguousarray(enc.col_counts, dtype=np.uint32)
        ro = np.ascontiguousarray(enc.row_offsets, dtype=np.uint32)
        co = np.ascontiguousarray(enc.col_offsets, dtype=np.uint32)
        pl = np.ascontiguousarray(enc.payload, dtype=np.float32)
        handle = _native._vp()
        grp = None if row_groups is None else np.ascontiguousarray(row_groups, dtype=np.int32)
        oo = None if out_order is None else np.ascontiguousarray(out_order, dtype=np.int32)
        _native.check(lib.tw_plan_create_cto_ex(
            ctypes_byref(handle), k, n, enc.config.granularity_g, rc.size,
            _native.ptr(rc, _native.ctypes.c_uint32), _native.ptr(cc, _native.ctypes.c_uint32),
            _native.ptr(ro, _native.ctypes.c_uint32), ro.shape[1],
            _native.ptr(co, _native.ctypes.c_uint32), co.shape[1],
            _native.ptr(pl, _native.ctypes.c_float), _DTYPE_CODES[self.compute_dtype],
            _native.SCHEDULES[schedule], 1 if row_layout == "runs" else 0,
            None if grp is None else _native.ptr(grp, _native.ctypes.c_int32),
            0 if grp is None else int(grp.size) - 1,
            None if oo is None else _native.ptr(oo, _native.ctypes.c_int32),
            _native.stream_handle()))
        self._handle = handle
        self._finalizer = weakref.finalize(self, lib.tw_plan_destroy, handle)
        self.per_tile_kept = [int(h) for h in rc]
        self.per_tile_width = [int(w) for w in cc]
        if overlay is not None:
            self.attach_overlay(overlay)
        self._refresh_info()

    @classmethod
    def from_cto1(cls, path, overlay: Optional[SparseOverlay] = None,
                  compute_dtype: str = "fp16", schedule: str = "lpt",
                  row_layout: str = "natural") -> "TwPlan":
        """Device plan straight from a CTO1 artifact: the file
        is read and validated like reference read_cto1 (formats.py:259-304)
        and the GPU weight format is built from it without re-pruning."""
        from .formats import read_cto1

        return cls(read_cto1(path), overlay, compute_dtype, schedule, row_layout)

    def save(self, path) -> int:
        """Write the device-native plan file "TWP1": the plan
        exactly as the kernels read it, so :meth:`load` skips the CTO
        validation, tile merging, row-run search and payload conversion.
        Returns the bytes written.  The overlay is not part of the file."""
        lib = _native.load_library()
        n = _native.ctypes.c_uint64(0)
        _native.check(lib.tw_plan_save(self._handle, None, _native.ctypes.byref(n)))
        buf = np.empty(int(n.value), dtype=np.uint8)
        _native.check(lib.tw_plan_save(self._handle, buf.ctypes.data, _native.ctypes.byref(n)))
        from pathlib import Path

        Path(path).write_bytes(buf.tobytes())
        return int(n.value)

    @classmethod
    def load(cls, path, overlay: Optional[SparseOverlay] = None) -> "TwPlan":
        """Plan from a "TWP1" file written by :meth:`save` (uploads only;
        every index is validated against the plan's dims by the library,
        CorruptEncodingError otherwise)."""
        from pathlib import Path

        torch = _torch()
        lib = _native.load_library()
        data = np.frombuffer(Path(path).read_bytes(), dtype=np.uint8)
        handle = _native._vp()
        _native.check(lib.tw_plan_load(ctypes_byref(handle), data.ctypes.data, data.size,
                                       _native.stream_handle()))
        self = cls.__new__(cls)
        self._handle = handle
        self._finalizer = weakref.finalize(self, lib.tw_plan_destroy, handle)
        self.device = torch.cuda.current_device()
        self._refresh_info()
        info = self.info
        self.compute_dtype = {_native.TW_F16: "fp16", _native.TW_BF16: "bf16",
                              _native.TW_F32: "fp32"}[info.compute_dtype]
        self.split = self.compute_dtype == "fp32"
        self.operand_dtype = "fp16" if self.split else self.compute_dtype
        self.schedule = "lpt"
        self.row_layout = "runs" if info.row_runs else "natural"
        self.original_dims = (int(info.k), int(info.n))
        self.per_tile_kept = []
        self.per_tile_width = []
        if overlay is not None:
            self.attach_overlay(overlay)
        return self

    # -- metadata -------------------------------------------------------
    def _refresh_info(self) -> None:
        lib = _native.load_library()
        info = _native.PlanInfo()
        _native.check(lib.tw_plan_get_info(self._handle, _native.ctypes.byref(info)))
        self.info = info
        cond = np.empty(info.n_condensed, dtype=np.int32)
        _native.check(lib.tw_plan_condensed_columns(self._handle,
                                                    _native.ptr(cond, _native.ctypes.c_int32)))
        uni = np.empty(info.n_union, dtype=np.int32)
        _native.check(lib.tw_plan_union_columns(self._handle,
                                                _native.ptr(uni, _native.ctypes.c_int32)))
        self.condensed_columns = cond.astype(np.int64)
        self.union_columns = uni.astype(np.int64)
        order = np.empty(info.k * max(1, info.row_copies), dtype=np.int32)
        _native.check(lib.tw_plan_row_order(self._handle, _native.ptr(order, _native.ctypes.c_int32)))
        self.row_order = order.astype(np.int64)  # layout position -> original K row
        self._row_order_dev = None
        self._masks = {}

    def column_mask(self, union: bool = False) -> IndexMask:
        """IndexMask of the output columns (condensed, or the TEW union),
        built once per plan (GemmOutput.column_map of every call)."""
        mk = self._masks.get(union)
        if mk is None:
            cols = self.union_columns if union else self.condensed_columns
            mk = IndexMask(self.original_dims[1], cols)
            self._masks[union] = mk
        return mk

    def output_groups(self) -> np.ndarray:
        """Ascending bounds of the C'^T row blocks each 128-column sub-tile
        writes (the groups a chained next plan's row layout may permute in)."""
        lib = _native.load_library()
        b = np.empty(int(self.info.n_sub) + 1, dtype=np.int32)
        _native.check(lib.tw_plan_output_groups(self._handle,
                                                _native.ptr(b, _native.ctypes.c_int32)))
        return b.astype(np.int64)

    @property
    def uses_row_runs(self) -> bool:
        """True when run()'s and run_tew()'s input is in this plan's permuted
        row layout (row_layout='runs' and the library found few-run row orders)."""
        return self.row_layout == "runs" and bool(self.info.row_runs)

    @property
    def has_overlay(self) -> bool:
        return bool(self.info.has_overlay)

    def attach_overlay(self, ov: SparseOverlay) -> None:
        if tuple(ov.dims) != tuple(self.original_dims):
            raise InvalidInputError(
                f"overlay dims {tuple(ov.dims)} do not match weights {tuple(self.original_dims)}")
        lib = _native.load_library()
        ptr_ = np.ascontiguousarray(ov.col_ptr, dtype=np.int64)
        rows = np.ascontiguousarray(ov.row_idx, dtype=np.int64)
        vals = np.ascontiguousarray(ov.values, dtype=np.float32)
        if rows.size == 0:
            rows = np.zeros(1, dtype=np.int64)
            vals = np.zeros(1, dtype=np.float32)
        k, n = self.original_dims
        _native.check(lib.tw_plan_attach_overlay(
            self._handle, k, n, int(ov.nnz), _native.ptr(ptr_, _native.ctypes.c_int64),
            _native.ptr(rows, _native.ctypes.c_int64), _native.ptr(vals, _native.ctypes.c_float),
            _native.stream_handle()))
        self._refresh_info()

    def set_sm_budget(self, sms: int) -> None:
        """Let K1 occupy at most ``sms`` SMs (0: all), so several plans
        launched on concurrent streams share the GPU (see TwPlanGroup)."""
        lib = _native.load_library()
        _native.check(lib.tw_plan_set_sm_budget(self._handle, int(sms)))
        self._refresh_info()

    def flops(self, m: int, tew: bool = False) -> int:
        """Surviving FLOPs of one product (metrics.py:114-117)."""
        macs = self.info.kept_macs_per_token if tew else self.info.kept_macs_per_token - self.info.nnz
        return 2 * int(m) * int(macs)

    # -- activations ------------------------------------------------------
    def prepare(self, a=None, *, at=None, stream=None, out=None):
        """Activations -> the A^T operand of :meth:`run` (K x M, compute dtype).

        ``a`` is the reference-layout activation matrix (M x K: numpy, nested
        list, CPU or CUDA tensor), transposed and cast on the GPU (K4) -- into
        the plan's permuted row order when :attr:`uses_row_runs`.
        Alternatively ``at`` is a CUDA A^T (K x M) in the original row order,
        returned as is when it already is the operand (compute dtype, unit
        token stride, token pitch a multiple of 8, 16-byte aligned base: the
        layout :meth:`run` writes, so one layer's output feeds the next), else
        copied (and row-permuted) into it.  ``out`` (with ``a``): a K x M
        CUDA view to write into.
        """
        torch = _torch()
        k = self.original_dims[0]
        if (a is None) == (at is None):
            raise InvalidInputError("pass exactly one of a (M x K) or at (K x M)")
        if a is not None:
            m_k = tuple(a.shape) if isinstance(a, torch.Tensor) else as_matrix(a).shape
            if len(m_k) != 2 or m_k[1] != k:
                raise InvalidInputError(
                    f"inner dims disagree: a has {m_k[-1]} cols, weights have K={k}")
            if not self.uses_row_runs and not self.split:
                return prepare_activations(a, self.compute_dtype, stream=stream, out=out)
            return self._prepare_runs(a, stream, out)
        if self.split:
            raise InvalidInputError("fp32 plans split A into fp16 hi / lo rows: pass a (M x K)")
        if not isinstance(at, torch.Tensor) or not at.is_cuda or at.dim() != 2:
            raise InvalidInputError("at must be a 2-D CUDA tensor (K x M)")
        if at.shape[0] != k:
            raise InvalidInputError(f"inner dims disagree: at has {at.shape[0]} rows, "
                                    f"weights have K={k}")
        if self.uses_row_runs:
            # the row permutation into the plan layout runs in the library
            # (tw_plan_permute_rows); a dtype cast, if needed, comes first
            if at.dtype != _torch_dtype(self.operand_dtype):
                at = at.to(_torch_dtype(self.operand_dtype))
            m = int(at.shape[1])
            if not _at_ready(at, self.operand_dtype):
                at = at.contiguous() if m % 8 == 0 else \
                    torch.nn.functional.pad(at, (0, (-m) % 8))[:, :m]
            rows = self.layout_rows
            ld = (m + 7) // 8 * 8
            x = torch.empty((rows, ld), dtype=at.dtype, device=at.device)
            lib = _native.load_library()
            _native.check(lib.tw_plan_permute_rows(
                self._handle, at.data_ptr(), m, at.stride(0) if at.shape[0] > 1 else ld,
                x.data_ptr(), ld, _native.stream_handle(stream)))
            return x[:, :m]
        if _at_ready(at, self.operand_dtype):
            return at
        # (after the row permutation at has layout_rows rows: row_copies x K)
        rows, m = int(at.shape[0]), int(at.shape[1])
        ld = (m + 7) // 8 * 8
        buf = torch.zeros((rows, ld), dtype=_torch_dtype(self.operand_dtype), device=at.device)
        buf[:, :m].copy_(at)
        return buf[:, :m]

    def _prepare_runs(self, a, stream, out):
        torch = _torch()
        k = self.original_dims[0]
        if isinstance(a, torch.Tensor):
            src = a if a.is_cuda else a.cuda(non_blocking=True)
            if src.dtype not in (torch.float32, torch.float16, torch.bfloat16):
                src = src.float()
            if src.stride(1) != 1:
                src = src.contiguous()
        else:
            src = torch.from_numpy(as_matrix(a)).cuda()
        m = int(src.shape[0])
        rows = self.layout_rows
        if out is not None:
            if tuple(out.shape) != (rows, m) or not _at_ready(out, self.operand_dtype):
                raise InvalidInputError(f"out must be a {rows} x M A^T view in the compute dtype")
            at, ld = out, out.stride(0)
        else:
            ld = (m + 7) // 8 * 8
            at = torch.empty((rows, ld), dtype=_torch_dtype(self.operand_dtype), device=src.device)
        lib = _native.load_library()
        _native.check(lib.tw_plan_prepare(self._handle, src.data_ptr(),
                                          _DTYPE_CODES[_dtype_name(src.dtype)], m, src.stride(0),
                                          at.data_ptr(), ld, _native.stream_handle(stream)))
        return at if out is not None else at[:, :m]

    # -- launches -------------------------------------------------------
    @property
    def layout_rows(self) -> int:
        """Rows of run()'s input: K, or row_copies x K in the row-run layout."""
        k = self.original_dims[0]
        return k * int(self.info.row_copies) if (self.uses_row_runs or self.split) else k

    def _check_x(self, x, rows=None):
        torch = _torch()
        if not isinstance(x, torch.Tensor) or not x.is_cuda:
            raise InvalidInputError("x must be a CUDA A^T (K x M) tensor, see TwPlan.prepare()")
        k = self.original_dims[0] if rows is None else rows
        if x.dim() != 2 or x.shape[0] != k:
            raise InvalidInputError(f"x must be {k} x M (plan layout rows x tokens), "
                                    f"got {tuple(x.shape)}")
        if x.dtype != _torch_dtype(self.operand_dtype):
            raise InvalidInputError(f"x dtype {x.dtype} != plan compute dtype "
                                    f"{self.operand_dtype}")
        if not _at_ready(x, self.operand_dtype):
            raise InvalidInputError("x must have unit token stride, a token pitch that is a "
                                    "multiple of 8 and a 16-byte aligned base "
                                    "(use TwPlan.prepare)")
        return int(x.shape[1]), int(x.stride(0)) if x.shape[0] > 1 else ((int(x.shape[1]) + 7) // 8 * 8)

    def _out(self, rows: int, m: int, out, out_dtype):
        """The C'^T output: a fresh (rows x M) tensor, or the caller's ``out``
        checked like the C ABI needs it (CUDA tensor on the plan's device,
        fp32/fp16/bf16, unit token stride, room for rows x M).  Misaligned
        views are allowed: the kernels fall back to narrower stores."""
        torch = _torch()
        if out is None:
            return torch.empty((rows, m), dtype=_torch_dtype(_dtype_name(out_dtype)),
                               device=f"cuda:{self.device}")
        if not isinstance(out, torch.Tensor) or not out.is_cuda:
            raise InvalidInputError("out must be a CUDA tensor")
        if out.device.index != self.device:
            raise InvalidInputError(f"out is on cuda:{out.device.index}, the plan on "
                                    f"cuda:{self.device}")
        if out.dtype not in (torch.float32, torch.float16, torch.bfloat16):
            raise InvalidInputError(f"out dtype {out.dtype} is not fp32/fp16/bf16")
        if out.dim() != 2 or out.shape[0] < rows or out.shape[1] < m or \
                (out.shape[1] > 1 and out.stride(1) != 1) or \
                (out.shape[0] > 1 and out.stride(0) < m):
            raise InvalidInputError("out must be a (rows x M) CUDA tensor with unit token stride")
        return out

    def run(self, x, out=None, out_dtype="fp32", stream=None, x_layout=None):
        """C'^T (N' x M) = TW product of x = A^T (K x M); K1 only.  x is in
        the plan's row layout: the original order for row_layout='natural',
        the permuted order :meth:`prepare` writes for row_layout='runs'
        (``x_layout='natural'`` overrides: original-order rows, gathered)."""
        if x_layout not in (None, "natural", "plan"):
            raise InvalidInputError(f"unknown x_layout {x_layout!r}")
        use_plan = self.uses_row_runs if x_layout is None else x_layout == "plan"
        if use_plan and not self.info.row_runs:
            raise InvalidInputError("this plan has no row-run layout")
        rows = self.layout_rows if (use_plan or self.split) else None
        m, ld = self._check_x(x, rows)
        ct = self._out(self.info.n_condensed, m, out, out_dtype)
        lib = _native.load_library()
        layout = _native.TW_LAYOUT_PLAN if use_plan else _native.TW_LAYOUT_NATURAL
        _native.check(lib.tw_gemm_ex(self._handle, x.data_ptr(), m, ld, ct.data_ptr(),
                                     ct.stride(0), _DTYPE_CODES[_dtype_name(ct.dtype)], layout,
                                     _native.stream_handle(stream)))
        return ct

    def run_tew(self, x, out=None, out_dtype="fp32", stream=None, x_layout=None):
        """C^T over the union columns (|union| x M) = TW + overlay; K1 + K2.
        K1 writes the condensed TW result to a scratch buffer (torch caching
        allocator, stream-ordered) that K2 scatters to the union rows.  x is
        in the plan's row layout, as for :meth:`run`."""
        if not self.has_overlay:
            raise InvalidInputError("plan has no overlay attached")
        if x_layout not in (None, "natural", "plan"):
            raise InvalidInputError(f"unknown x_layout {x_layout!r}")
        use_plan = self.uses_row_runs if x_layout is None else x_layout == "plan"
        if use_plan and not self.info.row_runs:
            raise InvalidInputError("this plan has no row-run layout")
        torch = _torch()
        m, ld = self._check_x(x, self.layout_rows if (use_plan or self.split) else None)
        ct = self._out(self.info.n_union, m, out, out_dtype)
        lib = _native.load_library()
        code = _DTYPE_CODES[_dtype_name(ct.dtype)]
        need = _native.ctypes.c_uint64()
        _native.check(lib.tw_plan_tew_workspace_bytes(self._handle, m, code,
                                                      _native.ctypes.byref(need)))
        ws = None
        if need.value:
            ws = torch.empty(int(need.value), dtype=torch.uint8, device=ct.device)
            if stream is not None:
                ws.record_stream(stream)  # freed by the caching allocator after K2 on `stream`
        layout = _native.TW_LAYOUT_PLAN if use_plan else _native.TW_LAYOUT_NATURAL
        _native.check(lib.tw_gemm_tew_ex(self._handle, x.data_ptr(), m, ld, ct.data_ptr(),
                                         ct.stride(0), code,
                                         ws.data_ptr() if ws is not None else None,
                                         int(need.value), layout, _native.stream_handle(stream)))
        return ct


    def run_tew_reuse(self, x, tile_ct, tile_columns=None, out=None, stream=None,
                      x_layout=None):
        """TEW result over the union columns from a tile product the caller
        already holds (K2 only: reference gemm_tew's ``tile_output``,
        executor.py:194).  ``tile_ct`` is the tile product as C^T rows (one row
        per output column, tokens contiguous) in the output dtype;
        ``tile_columns`` lists the original column of each of its rows (None:
        this plan's condensed columns).  Columns of the union missing from it
        start from zero, columns not in the union are dropped, exactly as
        ``expand()`` + re-condensing does in the reference."""
        if not self.has_overlay:
            raise InvalidInputError("plan has no overlay attached")
        if x_layout not in (None, "natural", "plan"):
            raise InvalidInputError(f"unknown x_layout {x_layout!r}")
        use_plan = self.uses_row_runs if x_layout is None else x_layout == "plan"
        torch = _torch()
        m, ld = self._check_x(x, self.layout_rows if (use_plan or self.split) else None)
        if not isinstance(tile_ct, torch.Tensor) or not tile_ct.is_cuda or tile_ct.dim() != 2 \
                or tile_ct.shape[1] != m or (m > 1 and tile_ct.stride(1) != 1):
            raise InvalidInputError("tile_ct must be a CUDA (columns x M) tensor with unit "
                                    "token stride")
        ct = self._out(self.info.n_union, m, out, _dtype_name(tile_ct.dtype))
        if ct.dtype != tile_ct.dtype:
            raise InvalidInputError("out and the tile product must share a dtype")
        rows_arg = None
        if tile_columns is not None:
            cols = np.asarray(tile_columns, dtype=np.int64)
            if cols.shape != (tile_ct.shape[0],):
                raise InvalidInputError("tile_columns must give one column per tile_ct row")
            pos = {int(c): i for i, c in enumerate(cols)}
            rows_arg = np.array([pos.get(int(u), -1) for u in self.union_columns],
                                dtype=np.int32)
        elif tile_ct.shape[0] != self.info.n_condensed:
            raise InvalidInputError(f"tile_ct has {tile_ct.shape[0]} rows, the plan "
                                    f"{self.info.n_condensed} condensed columns")
        ld_tile = int(tile_ct.stride(0)) if tile_ct.shape[0] > 1 else m
        lib = _native.load_library()
        layout = _native.TW_LAYOUT_PLAN if use_plan else _native.TW_LAYOUT_NATURAL
        _native.check(lib.tw_gemm_tew_reuse(
            self._handle, x.data_ptr(), m, ld, tile_ct.data_ptr(), ld_tile,
            None if rows_arg is None else _native.ptr(rows_arg, _native.ctypes.c_int32),
            ct.data_ptr(), ct.stride(0) if ct.shape[0] > 1 else m,
            _DTYPE_CODES[_dtype_name(ct.dtype)], layout, _native.stream_handle(stream)))
        return ct


def ctypes_byref(x):
    return _native.ctypes.byref(x)


def _at_ready(x, compute_dtype: str) -> bool:
    """x is usable as the A^T operand as is (see include/tw_gemm.h)."""
    if x.dtype != _torch_dtype(compute_dtype) or x.dim() != 2:
        return False
    if x.shape[1] > 1 and x.stride(1) != 1:
        return False
    pitch_ok = x.shape[0] == 1 or (x.stride(0) % 8 == 0 and x.stride(0) >= x.shape[1])
    return pitch_ok and x.data_ptr() % 16 == 0


def prepare_activations(a, compute_dtype: str = "fp16", stream=None, out=None):
    """Reference-layout activations (M x K) -> device A^T (K x M) in compute dtype.

    ``a`` may be a numpy array / nested list (coerced with :func:`as_matrix`
    like the reference, core.py:32-43) or a CUDA tensor.  The transpose and
    cast run in the K4 kernel; the token pitch is padded to a multiple of 8
    so rows stay 16-byte aligned.  Returns a K x M view (of ``out`` when
    given: a K x M CUDA view with unit token stride and a pitch that is a
    multiple of 8).
    """
    torch = _torch()
    cd = _dtype_name(compute_dtype)
    if isinstance(a, torch.Tensor):
        if a.dim() != 2 or a.shape[0] < 1 or a.shape[1] < 1:
            raise InvalidInputError(f"matrix must be 2-D with dims >= 1, got {tuple(a.shape)}")
        src = a if a.is_cuda else a.cuda(non_blocking=True)
        if src.dtype not in (torch.float32, torch.float16, torch.bfloat16):
            src = src.float()
        if src.stride(1) != 1:
            src = src.contiguous()
    else:
        src = torch.from_numpy(as_matrix(a)).cuda()
    m, k = src.shape
    if out is not None:
        if tuple(out.shape) != (k, m) or out.dtype != _torch_dtype(cd) or not _at_ready(out, cd):
            raise InvalidInputError("out must be a K x M A^T view in the compute dtype")
        at = out
        ld = out.stride(0) if k > 1 else (m + 7) // 8 * 8
    else:
        ld = (m + 7) // 8 * 8
        at = torch.empty((k, ld), dtype=_torch_dtype(cd), device=src.device)
    lib = _native.load_library()
    _native.check(lib.tw_transpose_cast(src.data_ptr(), _DTYPE_CODES[_dtype_name(src.dtype)], m,
                                        k, src.stride(0), at.data_ptr(), _DTYPE_CODES[cd], ld,
                                        _native.stream_handle(stream)))
    return at if out is not None else at[:, :m]


# ----------------------------------------------------------------------------
# plan cache keyed by the (immutable) reference objects
# ----------------------------------------------------------------------------

_PLAN_CACHE: dict = {}


def plan_for(b: Union[TileSparseMatrix, CtoEncoding], overlay: Optional[SparseOverlay] = None,
             compute_dtype: str = "fp16", schedule: str = "lpt",
             row_layout: str = "runs") -> TwPlan:
    """Cached :class:`TwPlan` for a tile matrix / encoding (+ overlay).

    The reference structures are frozen, so a plan is keyed by the identity
    of the objects it was built from and dropped when any of them dies.
    """
    torch = _torch()
    watched = [b] if overlay is None else [b, overlay]
    key = tuple(id(o) for o in watched) + (torch.cuda.current_device(), compute_dtype, schedule,
                                          row_layout)
    plan = _PLAN_CACHE.get(key)
    if plan is None:
        enc = b if isinstance(b, CtoEncoding) else encode_cto(b)
        plan = TwPlan(enc, overlay, compute_dtype, schedule, row_layout)
        _PLAN_CACHE[key] = plan
        for o in watched:
            weakref.finalize(o, _PLAN_CACHE.pop, key, None)
    return plan


# ----------------------------------------------------------------------------
# reference API
# ----------------------------------------------------------------------------

@dataclass
class GemmOutput:
    """Condensed product plus its column map (reference executor.py:68-80).

    ``condensed`` is an M x N_out CUDA tensor (a transposed view of the
    kernel's C'^T buffer, available as :attr:`condensed_t`).
    """

    condensed: object
    column_map: IndexMask

    @property
    def condensed_t(self):
        return self.condensed.t()

    def expand(self):
        """M x N CUDA tensor with zero columns at pruned positions."""
        torch = _torch()
        m = self.condensed.shape[0]
        out = torch.zeros((m, self.column_map.domain_len), dtype=self.condensed.dtype,
                          device=self.condensed.device)
        idx = torch.tensor(np.asarray(self.column_map.kept, dtype=np.int64), device=out.device)
        out.index_copy_(1, idx, self.condensed)
        return out

    def to_numpy(self) -> np.ndarray:
        """Condensed result on the host as float64 (the reference's carrier)."""
        return self.condensed.double().cpu().numpy()


@dataclass
class ExecutionTrace:
    """Per-tile work, assignment and balance (reference executor.py:83-118)."""

    strategy: str
    workers: int
    per_tile_macs: List[int]
    assignment: List[int]
    per_worker_macs: List[int]

    @property
    def total_macs(self) -> int:
        return int(sum(self.per_tile_macs))

    @property
    def total_flops(self) -> int:
        return 2 * self.total_macs

    @property
    def imbalance(self) -> float:
        t = np.asarray(self.per_worker_macs, dtype=np.float64)
        mean = t.mean()
        return float(t.max() / mean) if mean > 0 else 1.0

    def to_json_dict(self) -> dict:
        return {"strategy": self.strategy, "workers": self.workers,
                "per_tile_flops": [2 * v for v in self.per_tile_macs],
                "per_tile_macs": [int(v) for v in self.per_tile_macs],
                "assignment": [int(v) for v in self.assignment],
                "per_worker_flops": [2 * v for v in self.per_worker_macs],
                "imbalance": self.imbalance, "total_macs": self.total_macs,
                "total_flops": self.total_flops}


def schedule_tiles(per_tile_macs: List[int], workers: int, strategy: str = "lpt") -> List[int]:
    """Deterministic tile -> worker assignment (reference executor.py:206-227).

    ``lpt``: descending work onto the least-loaded worker (ties to the lower
    worker); ``round_robin``: tile i onto worker i % workers.
    """
    if workers < 1:
        raise InvalidInputError(f"workers must be >= 1, got {workers}")
    if strategy == "round_robin":
        return [i % workers for i in range(len(per_tile_macs))]
    if strategy != "lpt":
        raise InvalidInputError(f"unknown strategy {strategy!r}")
    loads = [0] * workers
    out = [0] * len(per_tile_macs)
    for i in sorted(range(len(per_tile_macs)), key=lambda t: (-per_tile_macs[t], t)):
        w = min(range(workers), key=lambda x: (loads[x], x))
        out[i] = w
        loads[w] += per_tile_macs[i]
    return out


def _activations(a, plan: "TwPlan"):
    """Reference-layout activations (M x K) -> the plan's A^T operand on the GPU."""
    return plan.prepare(a)


def gemm_tile_sparse(a, b: TileSparseMatrix, *, compute_dtype: str = "fp16",
                     out_dtype: str = "fp32") -> GemmOutput:
    """Per-tile gather + GEMM over every tile; output condensed to N'."""
    plan = plan_for(b, compute_dtype=compute_dtype)
    ct = plan.run(_activations(a, plan), out_dtype=out_dtype)
    return GemmOutput(condensed=ct.t(), column_map=b.column_mask)


def gemm_cto(a, c: CtoEncoding, check_padding: bool = False, *, compute_dtype: str = "fp16",
             out_dtype: str = "fp32") -> GemmOutput:
    """Single fused pass over the offset encoding.

    The library decodes and validates the offsets (CorruptEncodingError on
    malformed ones) and builds gather lists of exactly ``row_counts[i]``
    entries, so padded offsets are never dereferenced; ``check_padding`` is
    accepted for signature compatibility.
    """
    plan = plan_for(c, compute_dtype=compute_dtype)
    ct = plan.run(_activations(a, plan), out_dtype=out_dtype)
    return GemmOutput(condensed=ct.t(), column_map=plan.column_mask())


def execute_batched(a, b: TileSparseMatrix, workers: int, strategy: str = "lpt", *,
                    compute_dtype: str = "fp16",
                    out_dtype: str = "fp32") -> Tuple[GemmOutput, ExecutionTrace]:
    """All tiles in one persistent launch; ``strategy`` sets the sub-tile
    order inside each 128-token block (lpt = descending K').  The trace
    reports the reference's host-side LPT / round-robin assignment over
    ``workers`` lanes so accounting matches executor.py:241-265."""
    macs_per_token = [t.width * t.kept_rows.n_kept for t in b.tiles]
    assignment = schedule_tiles(macs_per_token, workers, strategy)
    plan = plan_for(b, compute_dtype=compute_dtype, schedule=strategy)
    x = _activations(a, plan)
    m = int(x.shape[1])
    ct = plan.run(x, out_dtype=out_dtype)
    per_tile = [m * v for v in macs_per_token]
    per_worker = [0] * workers
    for i, w in enumerate(assignment):
        per_worker[w] += per_tile[i]
    trace = ExecutionTrace(strategy=strategy, workers=workers, per_tile_macs=per_tile,
                           assignment=assignment, per_worker_macs=per_worker)
    return GemmOutput(condensed=ct.t(), column_map=b.column_mask), trace


def gemm_tew(a, b: TileSparseMatrix, ov: SparseOverlay,
             tile_output: Optional[GemmOutput] = None, *, compute_dtype: str = "fp16",
             out_dtype: str = "fp32") -> GemmOutput:
    """TW product + CSC overlay SpMM, condensed to the union of surviving
    columns (reference executor.py:180-203).  Without ``tile_output`` K1 and
    K2 run back to back; with it (the reference CLI's composition, cli.py:
    304-307) only K2 runs, on the caller's tile product, which is expanded
    to the original columns and re-condensed exactly as executor.py:194-203
    does (so a tile product that is not gemm_tile_sparse(a, b) is honoured)."""
    if tuple(ov.dims) != tuple(b.original_dims):
        raise InvalidInputError(f"overlay dims {tuple(ov.dims)} do not match weights "
                                f"{tuple(b.original_dims)}")
    plan = plan_for(b, overlay=ov, compute_dtype=compute_dtype)
    x = _activations(a, plan)
    if tile_output is None:
        ct = plan.run_tew(x, out_dtype=out_dtype)
    else:
        # reuse the caller's tile product (executor.py:194): K2 alone adds the
        # overlay onto it at the union columns
        cols = np.asarray(tile_output.column_map.kept, dtype=np.int64)
        same = cols.shape == plan.condensed_columns.shape and \
            np.array_equal(cols, plan.condensed_columns)
        ct = plan.run_tew_reuse(x, _tile_rows(tile_output, out_dtype),
                                tile_columns=None if same else cols)
    return GemmOutput(condensed=ct.t(), column_map=plan.column_mask(union=True))


def _tile_rows(out: "GemmOutput", out_dtype: str):
    """A GemmOutput's condensed M x N_t product as C^T rows (N_t x M, tokens
    contiguous) in ``out_dtype`` on the device: our own outputs already are
    (a transposed view), anything else goes through the K4 transpose-cast."""
    torch = _torch()
    cd = _dtype_name(out_dtype)
    c = out.condensed
    if isinstance(c, torch.Tensor) and c.is_cuda and c.dim() == 2 and \
            c.dtype == _torch_dtype(cd) and (c.shape[0] <= 1 or c.stride(0) == 1):
        return c.t()
    src = c if isinstance(c, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(c))
    if src.dim() != 2:
        raise InvalidInputError("tile_output.condensed must be 2-D (M x N_t)")
    src = src.cuda()
    if src.dtype not in (torch.float32, torch.float16, torch.bfloat16):
        src = src.float()
    if src.stride(1) != 1:
        src = src.contiguous()
    m, n_t = src.shape
    ld = max(1, m)
    rows = torch.empty((max(1, n_t), ld), dtype=_torch_dtype(cd), device=src.device)
    if m and n_t:
        lib = _native.load_library()
        _native.check(lib.tw_transpose_cast(src.data_ptr(), _DTYPE_CODES[_dtype_name(src.dtype)],
                                            m, n_t, src.stride(0), rows.data_ptr(),
                                            _DTYPE_CODES[cd], ld, _native.stream_handle()))
    return rows[:n_t, :m]


def gemm_dense(a, b):
    """Dense float64 product on the device (verification helper mirroring
    executor.py:40-65; cuBLAS DGEMM, not the reference's fixed k order)."""
    torch = _torch()
    a_t = torch.as_tensor(as_matrix(a) if not isinstance(a, torch.Tensor) else a).cuda().double()
    b_t = torch.as_tensor(as_matrix(b) if not isinstance(b, torch.Tensor) else b).cuda().double()
    if a_t.shape[1] != b_t.shape[0]:
        raise InvalidInputError(f"inner dims disagree: a is {tuple(a_t.shape)}, "
                                f"b is {tuple(b_t.shape)}")
    return a_t @ b_t


def masked_dense_reference(a, w, keep_mask: np.ndarray):
    """Zero pruned positions and run the dense float64 product on the device
    (verification helper mirroring executor.py:268-275)."""
    w = as_matrix(w)
    mask = np.asarray(keep_mask, dtype=bool)
    if mask.shape != w.shape:
        raise InvalidInputError(f"mask shape {mask.shape} != weights shape {w.shape}")
    return gemm_dense(a, np.where(mask, w, np.float32(0.0)))


def _as_f64(x) -> np.ndarray:
    try:
        import torch
        if isinstance(x, torch.Tensor):
            return x.detach().double().cpu().numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(x, dtype=ACC_DTYPE)


def relative_error(result, reference) -> float:
    """max|result - reference| / max|reference| (reference executor.py:278-288)."""
    r = _as_f64(result)
    ref = _as_f64(reference)
    if r.shape != ref.shape:
        raise InvalidInputError(f"shape mismatch: {r.shape} vs {ref.shape}")
    scale = float(np.max(np.abs(ref))) if ref.size else 0.0
    diff = float(np.max(np.abs(r - ref))) if r.size else 0.0
    if scale == 0.0:
        return 0.0 if diff == 0.0 else float("inf")
    return diff / scale


__all__ = ["TwPlan", "prepare_activations", "plan_for", "GemmOutput", "ExecutionTrace",
           "schedule_tiles", "gemm_tile_sparse", "gemm_cto", "execute_batched", "gemm_tew",
           "gemm_dense", "masked_dense_reference", "relative_error", "DeviceError"]
