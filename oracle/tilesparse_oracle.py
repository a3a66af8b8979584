"""TEST INFRASTRUCTURE ONLY -- restatement of the reference CPU path.

Every function cites the reference file:line it follows (paths relative to
/root/reference/pkg/src/tilesparse).  Parity status: pinned against the
golden vectors of tests/golden (generated from the reference itself).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor
from fractions import Fraction
from pathlib import Path
from typing import List, Sequence, Tuple

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_build" / "libtworacle.so"


# ----------------------------------------------------------------------------
# exact counting and naive pruning (small sizes only)
# ----------------------------------------------------------------------------

def floor_count(fraction: float, n: int) -> int:
    """core.py:46-60 -- floor(fraction*n) in rationals with a 2**-48 guard."""
    prod = Fraction(float(fraction)) * n
    base = math.floor(prod)
    if prod > 0 and (base + 1 - prod) <= prod / (1 << 48):
        return base + 1
    return base


def _rank_lowest(scores: Sequence[float], count: int) -> List[int]:
    """Units with the `count` lowest scores, ties to the lower id
    (core.py:158-160 rank_units)."""
    order = sorted(range(len(scores)), key=lambda i: (scores[i], i))
    return order[:count]


def naive_prune_tw(w: np.ndarray, s_t: float, g: int):
    """Plain-loop restatement of patterns.py:542-575 / tw_joint_prune 435-528.

    Column scores are sequential sums down each column (what numpy's
    sum(axis=0) does); segment scores use math.fsum so near-ties are not
    decided by summation order -- callers use data without such near-ties.
    Returns (keep_mask, kept_cols, [kept_rows per tile]).
    """
    w = np.asarray(w, dtype=np.float32)
    k, n = w.shape
    s = 1.0 - math.sqrt(1.0 - s_t)
    absw = [[abs(float(w[i, j])) for j in range(n)] for i in range(k)]
    col_scores = []
    for j in range(n):
        acc = 0.0
        for i in range(k):
            acc += absw[i][j]
        col_scores.append(acc)
    pruned = set(_rank_lowest(col_scores, floor_count(s, n)))
    if len(pruned) == n:  # min-keep clamp, patterns.py:462-468
        best = max(range(n), key=lambda j: (col_scores[j], -j))
        pruned.discard(best)
    kept_cols = [j for j in range(n) if j not in pruned]
    tiles = [kept_cols[t:t + g] for t in range(0, len(kept_cols), g)]
    seg_scores = []
    for cols in tiles:
        for r in range(k):
            seg_scores.append(math.fsum(absw[r][j] for j in cols))
    seg_pruned = set(_rank_lowest(seg_scores, floor_count(s, len(seg_scores))))
    rows_per_tile = []
    for t in range(len(tiles)):
        ids = [t * k + r for r in range(k)]
        if all(u in seg_pruned for u in ids):  # patterns.py:499-506
            best = max(ids, key=lambda u: (seg_scores[u], -u))
            seg_pruned.discard(best)
        rows_per_tile.append([r for r in range(k) if t * k + r not in seg_pruned])
    mask = np.zeros((k, n), dtype=bool)
    for cols, rows in zip(tiles, rows_per_tile):
        for r in rows:
            for j in cols:
                mask[r, j] = True
    return mask, kept_cols, rows_per_tile


def naive_tew_restore(w: np.ndarray, tw_mask: np.ndarray, delta: float):
    """patterns.py:578-602 -- restore floor(delta*K*N) best pruned elements,
    ties to the lowest flat index.  Returns the restored flat ids (sorted)."""
    k, n = w.shape
    flat = [abs(float(v)) for v in np.asarray(w, dtype=np.float32).ravel()]
    keep = tw_mask.ravel()
    cands = [i for i in range(k * n) if not keep[i]]
    count = min(floor_count(delta, k * n), len(cands))
    chosen = sorted(cands, key=lambda i: (-flat[i], i))[:count]
    return sorted(chosen)


# ----------------------------------------------------------------------------
# faithful numpy ports of the executor (CPU baseline timing)
# ----------------------------------------------------------------------------

def mac_kernel(a64: np.ndarray, b64: np.ndarray, out=None) -> np.ndarray:
    """executor.py:27-37 -- rank-1 update loop, strictly ascending k."""
    m, kk = a64.shape
    n = b64.shape[1]
    if out is None:
        out = np.zeros((m, n), dtype=np.float64)
    tmp = np.empty((m, n), dtype=np.float64)
    for i in range(kk):
        np.multiply(a64[:, i, None], b64[i, None, :], out=tmp)
        out += tmp
    return out


def tile_product(a64: np.ndarray, rows: np.ndarray, payload: np.ndarray) -> np.ndarray:
    """executor.py:121-124."""
    return mac_kernel(np.ascontiguousarray(a64[:, rows]),
                      np.ascontiguousarray(payload, dtype=np.float64))


def schedule_tiles(per_tile_macs: List[int], workers: int, strategy: str = "lpt") -> List[int]:
    """executor.py:206-227."""
    if strategy == "round_robin":
        return [i % workers for i in range(len(per_tile_macs))]
    loads = [0] * workers
    out = [0] * len(per_tile_macs)
    for i in sorted(range(len(per_tile_macs)), key=lambda t: (-per_tile_macs[t], t)):
        wk = min(range(workers), key=lambda x: (loads[x], x))
        out[i] = wk
        loads[wk] += per_tile_macs[i]
    return out


def execute_batched(a: np.ndarray, tiles: Sequence[Tuple[np.ndarray, np.ndarray]], workers: int,
                    strategy: str = "lpt") -> np.ndarray:
    """executor.py:230-265 -- tiles = [(kept_rows, payload K'xw)], lanes write
    disjoint column ranges; returns the condensed fp64 output."""
    a64 = np.asarray(a, dtype=np.float32).astype(np.float64)
    m = a64.shape[0]
    widths = [p.shape[1] for _, p in tiles]
    macs = [m * p.shape[1] * p.shape[0] for _, p in tiles]
    assignment = schedule_tiles(macs, workers, strategy)
    starts = np.concatenate([[0], np.cumsum(widths)]).astype(np.int64)
    out = np.empty((m, int(starts[-1])), dtype=np.float64)

    def lane(wk: int) -> None:
        for i, (rows, p) in enumerate(tiles):
            if assignment[i] == wk:
                out[:, starts[i]:starts[i + 1]] = tile_product(a64, rows, p)

    if workers == 1:
        lane(0)
    else:
        with ThreadPoolExecutor(max_workers=workers) as pool:
            list(pool.map(lane, range(workers)))
    return out


def gemm_tew_add(a: np.ndarray, full: np.ndarray, col_ptr, row_idx, values) -> np.ndarray:
    """executor.py:197-200 -- add the overlay columns into an expanded output."""
    a64 = np.asarray(a, dtype=np.float32).astype(np.float64)
    for c in np.flatnonzero(np.diff(col_ptr)):
        lo, hi = int(col_ptr[c]), int(col_ptr[c + 1])
        full[:, c] += a64[:, row_idx[lo:hi]] @ np.asarray(values[lo:hi], dtype=np.float64)
    return full


# ----------------------------------------------------------------------------
# C oracle (tw_oracle.c)
# ----------------------------------------------------------------------------

_lib = None


def build_c_oracle(force: bool = False) -> Path:
    src = HERE / "tw_oracle.c"
    if force or not LIB_PATH.exists() or LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


def _load():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build_c_oracle()
        lib = ctypes.CDLL(str(LIB_PATH))
        u32p = ctypes.POINTER(ctypes.c_uint32)
        lib.tw_oracle_gemm_cto.argtypes = [
            ctypes.POINTER(ctypes.c_float), ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
            u32p, u32p, u32p, ctypes.c_int32, u32p, ctypes.c_int32,
            ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_double), ctypes.c_int32]
        lib.tw_oracle_overlay_add.argtypes = [
            ctypes.POINTER(ctypes.c_float), ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
            ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64),
            ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_double)]
        _lib = lib
    return _lib


def _p(arr, ct):
    return arr.ctypes.data_as(ctypes.POINTER(ct))


def c_gemm_cto(a: np.ndarray, row_counts, col_counts, row_offsets, col_offsets, payload,
               threads: int = 0) -> np.ndarray:
    """Condensed fp64 product of a CTO encoding (bit-exact with gemm_cto)."""
    lib = _load()
    a = np.ascontiguousarray(a, dtype=np.float32)
    rc = np.ascontiguousarray(row_counts, dtype=np.uint32)
    cc = np.ascontiguousarray(col_counts, dtype=np.uint32)
    ro = np.ascontiguousarray(row_offsets, dtype=np.uint32)
    co = np.ascontiguousarray(col_offsets, dtype=np.uint32)
    pl = np.ascontiguousarray(payload, dtype=np.float32)
    m, k = a.shape
    out = np.empty((m, int(cc.sum())), dtype=np.float64)
    threads = threads or (os.cpu_count() or 1)
    rc_ = lib.tw_oracle_gemm_cto(_p(a, ctypes.c_float), m, k, rc.size, _p(rc, ctypes.c_uint32),
                                 _p(cc, ctypes.c_uint32), _p(ro, ctypes.c_uint32), ro.shape[1],
                                 _p(co, ctypes.c_uint32), co.shape[1], _p(pl, ctypes.c_float),
                                 _p(out, ctypes.c_double), threads)
    if rc_:
        raise RuntimeError("oracle allocation failed")
    return out


def c_gemm_cto_enc(a: np.ndarray, enc, threads: int = 0) -> np.ndarray:
    return c_gemm_cto(a, enc.row_counts, enc.col_counts, enc.row_offsets, enc.col_offsets,
                      enc.payload, threads)


def c_overlay_add(a: np.ndarray, full: np.ndarray, col_ptr, row_idx, values) -> np.ndarray:
    lib = _load()
    a = np.ascontiguousarray(a, dtype=np.float32)
    full = np.ascontiguousarray(full, dtype=np.float64)
    cp = np.ascontiguousarray(col_ptr, dtype=np.int64)
    ri = np.ascontiguousarray(row_idx, dtype=np.int64)
    va = np.ascontiguousarray(values, dtype=np.float32)
    if ri.size == 0:
        return full
    m, k = a.shape
    lib.tw_oracle_overlay_add(_p(a, ctypes.c_float), m, k, full.shape[1],
                              _p(cp, ctypes.c_int64), _p(ri, ctypes.c_int64),
                              _p(va, ctypes.c_float), _p(full, ctypes.c_double))
    return full


def tew_reference(a: np.ndarray, enc, col_ptr, row_idx, values, n: int):
    """TEW output restricted to the union columns (executor.py:194-203):
    returns (condensed fp64 M x |union|, union column ids)."""
    cond = c_gemm_cto_enc(a, enc)
    kept_cols = []
    for i in range(enc.row_counts.size):
        w = int(enc.col_counts[i])
        kept_cols.append(np.arange(w, dtype=np.int64) + enc.col_offsets[i, :w].astype(np.int64))
    kept_cols = np.concatenate(kept_cols)
    full = np.zeros((a.shape[0], n), dtype=np.float64)
    full[:, kept_cols] = cond
    full = c_overlay_add(a, full, col_ptr, row_idx, values)
    ov_cols = np.flatnonzero(np.diff(np.asarray(col_ptr)))
    union = np.union1d(kept_cols, ov_cols)
    return np.ascontiguousarray(full[:, union]), union
