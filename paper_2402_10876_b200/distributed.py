"""Multi-GPU driver (K5): one process per GPU over torch.distributed / NCCL.

Two ways the TW path shards:

* **column tiles** (large layers, config 5): tiles own disjoint output
  columns (executor.py:233-236 -- each column range is written by exactly
  one tile), so rank r keeps a contiguous group of tiles, computes its rows
  of C'^T, and one ``all_gather_into_tensor`` assembles C'^T.  Because the
  native output is C'^T (one row per output column, tokens contiguous), each
  rank's shard is a contiguous row block: no permute before or after the
  collective.
* **token (M) split** (small layers, BERT / VGG): every rank holds the full
  weight and an M/P slice of tokens; outputs stay sharded, no collective.

The partition logic is pure host code and is tested on CPU with gloo
(tests/test_distributed.py); the GPU product path uses the same functions
with the sm_100a kernel on each rank and NCCL for the gather.
"""

from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np

from .errors import InvalidInputError
from .formats import CtoEncoding


def partition_contiguous(costs: Sequence[int], parts: int) -> List[Tuple[int, int]]:
    """Split items 0..n-1 into ``parts`` contiguous [lo, hi) ranges with
    near-equal cost (greedy prefix cut at the running ideal share).  Ranges
    may be empty when parts > n."""
    n = len(costs)
    if parts < 1:
        raise InvalidInputError(f"parts must be >= 1, got {parts}")
    total = float(sum(costs))
    bounds, lo, acc = [], 0, 0.0
    prefix = np.concatenate([[0.0], np.cumsum(np.asarray(costs, dtype=np.float64))])
    for p in range(parts):
        if p == parts - 1:
            hi = n
        else:
            target = total * (p + 1) / parts
            # first index whose prefix reaches the target, at least lo
            hi = int(np.searchsorted(prefix, target, side="left"))
            hi = min(max(hi, lo), n)
            # choose the closer of hi-1 / hi to the target
            if hi > lo and abs(prefix[hi - 1] - target) < abs(prefix[hi] - target):
                hi -= 1
        bounds.append((lo, hi))
        lo = hi
    del acc
    return bounds


def shard_encoding(enc: CtoEncoding, lo: int, hi: int) -> CtoEncoding:
    """Sub-encoding holding tiles [lo, hi) of ``enc`` (same K, N, g; column
    offsets keep their original column ids)."""
    if not 0 <= lo < hi <= enc.tile_count:
        raise InvalidInputError(f"bad tile range [{lo}, {hi}) of {enc.tile_count}")
    b = enc.payload_bounds()
    return CtoEncoding(original_dims=enc.original_dims, config=enc.config,
                       row_counts=enc.row_counts[lo:hi], col_counts=enc.col_counts[lo:hi],
                       row_offsets=enc.row_offsets[lo:hi], col_offsets=enc.col_offsets[lo:hi],
                       payload=enc.payload[b[lo]:b[hi]])


def column_shards(enc: CtoEncoding, world: int) -> List[Tuple[int, int]]:
    """Contiguous tile ranges per rank, balanced by surviving MACs."""
    macs = (enc.row_counts.astype(np.int64) * enc.col_counts.astype(np.int64)).tolist()
    return partition_contiguous(macs, world)


def shard_rows(enc: CtoEncoding, shards: Sequence[Tuple[int, int]]) -> List[Tuple[int, int]]:
    """Condensed output row range [lo, hi) of C'^T owned by every shard."""
    starts = np.concatenate([[0], np.cumsum(enc.col_counts.astype(np.int64))])
    return [(int(starts[lo]), int(starts[hi])) for lo, hi in shards]


def token_slice(m: int, world: int, rank: int) -> Tuple[int, int]:
    """[lo, hi) token range of ``rank`` for the M-split (multiples of 128
    tokens except the tail, so every rank runs whole 128-token blocks)."""
    blocks = -(-m // 128)
    lo_b = blocks * rank // world
    hi_b = blocks * (rank + 1) // world
    return min(lo_b * 128, m), min(hi_b * 128, m)


def gather_rows(local, rows: Sequence[Tuple[int, int]], group=None):
    """All-gather row shards of C'^T into the full (sum rows) x M tensor.

    ``local`` is this rank's (hi - lo) x M shard.  Shards of unequal height
    are padded to the tallest one for ``all_gather_into_tensor`` and the
    padding is sliced away; equal shards gather with no extra copy.
    """
    import torch
    import torch.distributed as dist

    heights = [hi - lo for lo, hi in rows]
    tallest = max(heights)
    m = local.shape[1]
    world = len(rows)
    if all(h == tallest for h in heights):
        out = torch.empty((tallest * world, m), dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(out, local.contiguous(), group=group)
        return out
    padded = torch.zeros((tallest, m), dtype=local.dtype, device=local.device)
    padded[:local.shape[0]].copy_(local)
    buf = torch.empty((tallest * world, m), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(buf, padded, group=group)
    parts = [buf[r * tallest:r * tallest + heights[r]] for r in range(world)]
    return torch.cat(parts, dim=0)
