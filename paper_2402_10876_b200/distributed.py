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


def token_chunks(m: int, chunks: int, align: int = 256) -> List[Tuple[int, int]]:
    """[lo, hi) token ranges of ``chunks`` near-equal pieces of M on
    ``align``-token boundaries (whole K1 units; the last piece takes the tail)."""
    if chunks < 1:
        raise InvalidInputError(f"chunks must be >= 1, got {chunks}")
    units = -(-m // align)
    chunks = max(1, min(chunks, units))
    out = []
    for j in range(chunks):
        lo = min(m, units * j // chunks * align)
        hi = min(m, units * (j + 1) // chunks * align)
        out.append((lo, hi))
    return out


class ChunkedRows:
    """An all-gathered C'^T stored token-chunk-major: ``parts[j]`` is the
    full (N' x M_j) C'^T of token chunk j.  TW layers act on every token
    independently, so each part is a complete A^T for the next layer's
    tokens of that chunk; :meth:`full` assembles the (N' x M) tensor."""

    def __init__(self, parts, spans):
        self.parts = parts
        self.spans = spans

    @property
    def shape(self):
        return (int(self.parts[0].shape[0]), int(self.spans[-1][1]))

    def full(self):
        import torch

        if len(self.parts) == 1:
            return self.parts[0]
        return torch.cat(self.parts, dim=1)


class TwShardedPlan:
    """One TW layer sharded over the ranks of a process group by column tiles
    (configs[4]).

    Tiles own disjoint output columns (reference executor.py:233-236), so
    rank r keeps a contiguous, MAC-balanced group of tiles
    (:func:`column_shards`), runs K1 on it and the ranks all-gather their
    rows of C'^T -- contiguous row blocks of the native layout, so the
    collective needs no permute.  With ``chunks > 1`` the tokens are cut into
    M-chunks: the all-gather of chunk j (NCCL's stream, ``async_op``)
    overlaps K1 of chunk j + 1 on the compute stream, and the result is a
    :class:`ChunkedRows`.  Every rank holds the full A^T (replicated input).

    ``local_product(x, out)`` replaces the per-rank product (tests on CPU
    ranks); by default it is this rank's :class:`TwPlan` (the sm_100a path).
    """

    def __init__(self, enc: CtoEncoding, group=None, *, compute_dtype: str = "fp16",
                 row_layout: str = "natural", chunks: int = 1, local_product=None):
        import torch.distributed as dist

        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.shards = column_shards(enc, self.world)
        self.rows = shard_rows(enc, self.shards)
        self.heights = [hi - lo for lo, hi in self.rows]
        self.tallest = max(self.heights)
        self.n_condensed = int(sum(self.heights))
        self.original_dims = enc.original_dims
        self.chunks = int(chunks)
        if self.chunks < 1:
            raise InvalidInputError(f"chunks must be >= 1, got {chunks}")
        starts = np.concatenate([[0], np.cumsum(enc.col_counts.astype(np.int64))])
        cols = []
        for i in range(enc.tile_count):
            w = int(enc.col_counts[i])
            cols.append(np.arange(w, dtype=np.int64) + enc.col_offsets[i, :w].astype(np.int64))
        self.condensed_columns = np.concatenate(cols) if cols else np.zeros(0, np.int64)
        assert self.condensed_columns.size == int(starts[-1])
        lo, hi = self.shards[self.rank]
        self.plan = None
        self._local = local_product
        if local_product is None and hi > lo:
            from .executor import TwPlan

            self.plan = TwPlan(shard_encoding(enc, lo, hi), compute_dtype=compute_dtype,
                               row_layout=row_layout)
        self.compute_dtype = compute_dtype

    def prepare(self, a=None, *, at=None):
        """A (M x K) or a natural-order A^T -> this rank's plan operand."""
        if self.plan is not None:
            return self.plan.prepare(a, at=at)
        if at is not None:
            return at
        from .executor import prepare_activations

        return prepare_activations(a, self.compute_dtype)

    def _product(self, x, out):
        if self._local is not None:
            self._local(x, out)
        elif self.plan is not None:
            self.plan.run(x, out=out)

    def _gather(self, local, async_op=False):
        """all_gather_into_tensor of the (tallest x m) row shards."""
        import torch
        import torch.distributed as dist

        m = local.shape[1]
        buf = torch.empty((self.tallest * self.world, m), dtype=local.dtype, device=local.device)
        if self.world == 1:
            buf.copy_(local)
            return buf, None
        if local.is_cuda and dist.get_backend(self.group) != "nccl":
            # a host-only backend (gloo, e.g. ranks sharing one GPU): stage on the host
            host = torch.empty((self.tallest * self.world, m), dtype=local.dtype)
            dist.all_gather_into_tensor(host, local.cpu(), group=self.group)
            buf.copy_(host)
            return buf, None
        work = dist.all_gather_into_tensor(buf, local, group=self.group, async_op=async_op)
        return buf, work

    def _compact(self, buf):
        """(world x tallest) x m gathered rows -> N' x m (drops shard padding)."""
        import torch

        if all(h == self.tallest for h in self.heights):
            return buf
        return torch.cat([buf[r * self.tallest:r * self.tallest + h]
                          for r, h in enumerate(self.heights)], dim=0)

    def run(self, x, out_dtype: str = "fp16"):
        """Full C'^T of the layer on every rank: (N' x M) for chunks == 1,
        else a :class:`ChunkedRows` of the M-chunks."""
        import torch

        dt = {"fp32": torch.float32, "fp16": torch.float16, "bf16": torch.bfloat16}.get(out_dtype)
        if dt is None:
            raise InvalidInputError(f"unknown out_dtype {out_dtype!r}")
        m = int(x.shape[1])
        spans = token_chunks(m, self.chunks)
        h = self.heights[self.rank]
        parts, works = [], []
        for lo, hi in spans:
            local = torch.zeros((self.tallest, hi - lo), dtype=dt, device=x.device) \
                if h < self.tallest else torch.empty((self.tallest, hi - lo), dtype=dt,
                                                     device=x.device)
            if h:
                self._product(x[:, lo:hi], local[:h])
            buf, work = self._gather(local, async_op=len(spans) > 1)
            parts.append(buf)
            works.append(work)
        for w in works:
            if w is not None:
                w.wait()
        parts = [self._compact(p) for p in parts]
        if len(parts) == 1:
            return parts[0]
        return ChunkedRows(parts, spans)
