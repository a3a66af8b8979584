"""FLOP accounting for the TW/TEW matmul.

Restates the FLOP definition of reference metrics.py:105-147, which is the
denominator of every "effective TFLOP/s" this framework reports:

    sparse_flops = 2 * M * sum_i(width_i * kept_rows_i) + 2 * M * overlay_nnz
    dense_flops  = 2 * M * K * N

The reference's CPU memory model (u16 offsets vs byte masks, metrics.py
:122-135) is kept only for the payload/index byte counts; the GPU roofline
byte model lives in :func:`algorithmic_bytes`.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Optional

from .errors import InvalidInputError
from .patterns import PrunePlan, SparseOverlay, TileSparseMatrix

REPORT_SCHEMA = "report-v1"


@dataclass
class SparsityReport:
    pattern: str
    target: float
    achieved: float
    m_rows: int
    dense_flops: int
    sparse_flops: int
    flop_reduction: float
    imbalance: float
    per_tile_flops: List[int]
    memory: Dict[str, int]

    def to_json_dict(self) -> dict:
        return {"schema": REPORT_SCHEMA, "pattern": self.pattern, "target": float(self.target),
                "achieved": float(self.achieved), "m_rows": int(self.m_rows),
                "dense_flops": int(self.dense_flops), "sparse_flops": int(self.sparse_flops),
                "flop_reduction": float(self.flop_reduction), "imbalance": float(self.imbalance),
                "per_tile_flops": [int(v) for v in self.per_tile_flops],
                "memory": {k: int(v) for k, v in self.memory.items()}}


def tile_flops(tsm: TileSparseMatrix, m_rows: int) -> List[int]:
    """2 * M * width * kept_rows per tile (metrics.py:114)."""
    return [2 * m_rows * t.width * t.kept_rows.n_kept for t in tsm.tiles]


def sparse_flops(tsm: TileSparseMatrix, m_rows: int,
                 overlay: Optional[SparseOverlay] = None) -> int:
    """Surviving FLOPs of one product (metrics.py:114-117)."""
    extra = 2 * m_rows * overlay.nnz if overlay is not None else 0
    return sum(tile_flops(tsm, m_rows)) + extra


def report(plan: PrunePlan, tsm: TileSparseMatrix, m_rows: int,
           overlay: Optional[SparseOverlay] = None) -> SparsityReport:
    """Account one pruned matrix for a GEMM with ``m_rows`` input rows."""
    if m_rows < 1:
        raise InvalidInputError(f"m_rows must be >= 1, got {m_rows}")
    if not isinstance(tsm, TileSparseMatrix):
        raise InvalidInputError("report() on this path takes a TileSparseMatrix")
    k, n = tsm.original_dims
    if (k, n) != tuple(plan.shape):
        raise InvalidInputError(
            f"plan shape {tuple(plan.shape)} does not match representation {(k, n)}")
    per_tile = tile_flops(tsm, m_rows)
    total = sparse_flops(tsm, m_rows, overlay)
    dense = 2 * m_rows * k * n
    mean = sum(per_tile) / len(per_tile)
    memory = {"dense_bytes": 4 * k * n,
              "payload_bytes": 4 * sum(t.width * t.kept_rows.n_kept for t in tsm.tiles),
              "index_bytes": 2 * sum(t.width + t.kept_rows.n_kept for t in tsm.tiles)}
    memory["total_sparse_bytes"] = memory["payload_bytes"] + memory["index_bytes"]
    if overlay is not None:
        memory["overlay_bytes"] = overlay.nnz * 6 + (n + 1) * 4
        memory["total_sparse_bytes"] += memory["overlay_bytes"]
    return SparsityReport(pattern=plan.pattern, target=plan.target_sparsity,
                          achieved=plan.achieved_sparsity, m_rows=m_rows, dense_flops=dense,
                          sparse_flops=total, flop_reduction=1.0 - total / dense,
                          imbalance=(max(per_tile) / mean) if mean > 0 else 1.0,
                          per_tile_flops=per_tile, memory=memory)


def algorithmic_bytes(tsm: TileSparseMatrix, m_rows: int, e_in: int = 2, e_w: int = 2,
                      e_out: int = 2, overlay: Optional[SparseOverlay] = None,
                      n_out: Optional[int] = None) -> int:
    """Compulsory HBM bytes of one GPU launch:

    A read once (M*K), payload + row indices read once, output written once,
    plus overlay values / rows / column pointers for TEW.
    """
    k, n = tsm.original_dims
    kept = sum(t.width * t.kept_rows.n_kept for t in tsm.tiles)
    rows = sum(t.kept_rows.n_kept for t in tsm.tiles)
    if n_out is None:
        n_out = tsm.n_condensed
    total = e_in * m_rows * k + e_w * kept + 4 * rows + e_out * m_rows * n_out
    if overlay is not None:
        total += (e_w + 4) * overlay.nnz + 4 * (n + 1)
    return int(total)
