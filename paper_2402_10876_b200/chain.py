"""Layer chaining in the native layout.

K1 writes C'^T: one row per *kept* output column of layer l, tokens
contiguous.  That is already the A^T layout the next layer reads, except
that its rows are the N'_l condensed columns rather than all N_l.  The
reference would feed layer l+1 the expanded M x N_l output
(``GemmOutput.expand``, executor.py:75-80), whose pruned columns are exact
zeros, so every kept row of layer l+1 that falls on a column pruned by layer l
contributes exactly 0 (executor.py:27-37 adds a * 0 terms).

:func:`chain_encoding` rewrites layer l+1's CTO encoding (formats.py:82-181)
into the condensed row space of layer l: kept rows on pruned columns are
dropped (with their payload entries) and the survivors are renumbered by
their position in layer l's ``column_mask``.  The chained plan then consumes
layer l's C'^T buffer directly -- no expand, no transpose, no copy -- and
does only the MACs whose inputs can be non-zero.  It is exact whenever the
map between the layers sends 0 to 0 (a plain product chain, ReLU / GELU
without a bias on pruned columns).
"""

from __future__ import annotations

import numpy as np

from .core import TileConfig
from .errors import InvalidInputError
from .formats import PAD_SENTINEL, CtoEncoding


def chain_encoding(enc_next: CtoEncoding, prev_columns) -> CtoEncoding:
    """Encoding of layer l+1 over the condensed output rows of layer l.

    ``prev_columns`` is layer l's kept column ids (``column_mask.kept`` or
    ``TwPlan.condensed_columns``), strictly increasing within
    ``[0, enc_next.original_dims[0])``.  A tile whose kept rows all fall on
    pruned columns keeps one zero-payload row (every tile keeps >= 1 row,
    formats.py:94-127), so its output columns are exact zeros.
    """
    prev = np.asarray(prev_columns, dtype=np.int64)
    k_next, n_next = enc_next.original_dims
    if prev.ndim != 1 or prev.size < 1:
        raise InvalidInputError("prev_columns must be a non-empty 1-D index list")
    if prev[0] < 0 or prev[-1] >= k_next or np.any(prev[1:] <= prev[:-1]):
        raise InvalidInputError(
            f"prev_columns must be strictly increasing within [0, {k_next}) "
            "(the next layer's input dimension)")
    pos = np.full(k_next, -1, dtype=np.int64)
    pos[prev] = np.arange(prev.size)
    rows_out, payload_out = [], []
    for i in range(enc_next.tile_count):
        rows = enc_next.tile_rows(i)
        pt = enc_next.tile_payload_t(i)            # width x kept rows
        live = pos[rows] >= 0
        if live.any():
            rows_out.append(pos[rows[live]])
            payload_out.append(np.ascontiguousarray(pt[:, live]))
        else:
            rows_out.append(np.zeros(1, dtype=np.int64))
            payload_out.append(np.zeros((pt.shape[0], 1), dtype=pt.dtype))
    rc = np.array([r.size for r in rows_out], dtype=np.uint32)
    ro = np.full((rc.size, int(rc.max())), PAD_SENTINEL, dtype=np.uint32)
    for i, r in enumerate(rows_out):
        ro[i, :r.size] = r - np.arange(r.size)
    return CtoEncoding(original_dims=(int(prev.size), n_next),
                       config=TileConfig(granularity_g=enc_next.config.granularity_g,
                                         input_tile_t=enc_next.config.input_tile_t),
                       row_counts=rc, col_counts=enc_next.col_counts,
                       row_offsets=ro, col_offsets=enc_next.col_offsets,
                       payload=np.concatenate([p.ravel() for p in payload_out]))


def chain_plans(enc_prev: CtoEncoding, enc_next: CtoEncoding, compute_dtype: str = "fp16"):
    """Two device plans for layer l -> layer l+1 in the row-run layout.

    Layer l+1 is re-encoded over layer l's condensed output rows
    (:func:`chain_encoding`) and gets a row-run layout whose permutation stays
    inside each 128-row block that one of layer l's sub-tiles writes; layer l
    is then built with that permutation as its output row order (payload rows
    reordered inside each sub-tile, so its TMA-store epilogue is unchanged).
    Layer l's C'^T is therefore already layer l+1's plan-layout A^T: the
    second product reads it with dense TMA boxes, with no prepare / permute
    pass between them.  Returns ``(prev, next)``; ``prev.condensed_columns``
    lists the original column of each of its output rows in that order.
    """
    from .executor import TwPlan

    probe = TwPlan(enc_prev, compute_dtype=compute_dtype)
    groups = probe.output_groups()
    cols = probe.condensed_columns
    del probe
    chained = chain_encoding(enc_next, cols)
    nxt = TwPlan(chained, compute_dtype=compute_dtype, row_layout="runs", row_groups=groups)
    if nxt.uses_row_runs:
        order = np.empty(nxt.row_order.size, dtype=np.int64)
        order[nxt.row_order] = np.arange(nxt.row_order.size)   # condensed col -> position
        prev = TwPlan(enc_prev, compute_dtype=compute_dtype, out_order=order)
    else:
        prev = TwPlan(enc_prev, compute_dtype=compute_dtype)
    return prev, nxt


__all__ = ["chain_encoding", "chain_plans"]
