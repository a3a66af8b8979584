"""Multi-rank partition logic on CPU (gloo, world_size 2).

The GPU path runs the sm_100a kernel per rank and NCCL for the gather; here
each rank computes its shard with the CPU oracle so the partition, the
contiguous C'^T row ownership and the all-gather assembly are checked
without a GPU.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import paper_2402_10876_b200 as tw
from paper_2402_10876_b200 import distributed as D


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem():
    rng = np.random.default_rng(42)
    w = rng.normal(size=(96, 200)).astype(np.float32)
    a = rng.normal(size=(50, 96)).astype(np.float32)
    _, tsm = tw.prune_tw(w, 0.5, 16)
    return a, tw.encode_cto(tsm)


def _worker(rank, world, port, mode, results):
    import torch
    import torch.distributed as dist

    from oracle import tilesparse_oracle as orc

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a, enc = _problem()
        if mode == "columns":
            shards = D.column_shards(enc, world)
            rows = D.shard_rows(enc, shards)
            lo, hi = shards[rank]
            sub = D.shard_encoding(enc, lo, hi)
            local = torch.from_numpy(np.ascontiguousarray(orc.c_gemm_cto_enc(a, sub).T))
            full_t = D.gather_rows(local, rows)
            results[rank] = full_t.numpy().T.copy()
        else:
            m = a.shape[0]
            spans = [D.token_slice(m, world, r) for r in range(world)]
            lo, hi = spans[rank]
            local = torch.from_numpy(orc.c_gemm_cto_enc(a[lo:hi], enc))
            tallest = max(h - l for l, h in spans)
            pad = torch.zeros((tallest, local.shape[1]), dtype=local.dtype)
            pad[:hi - lo] = local
            bufs = [torch.empty_like(pad) for _ in range(world)]
            dist.all_gather(bufs, pad)
            results[rank] = np.concatenate([bufs[r][:h - l].numpy()
                                            for r, (l, h) in enumerate(spans)])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["columns", "tokens"])
def test_two_rank_sharding_equals_single_device(mode):
    from oracle import tilesparse_oracle as orc

    a, enc = _problem()
    want = orc.c_gemm_cto_enc(a, enc)
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), mode, results), nprocs=2, join=True)
    for r in range(2):
        assert np.array_equal(results[r], want)


def test_partition_contiguous_balances():
    bounds = D.partition_contiguous([10] * 64, 8)
    assert bounds == [(8 * i, 8 * i + 8) for i in range(8)]
    b = D.partition_contiguous([100, 1, 1, 1, 1, 100], 2)
    assert b == [(0, 3), (3, 6)]
    b = D.partition_contiguous([5, 5], 4)
    assert b[-1][1] == 2 and sum(hi - lo for lo, hi in b) == 2


def test_token_slice_covers_m():
    for m in (1, 127, 128, 1000, 8192):
        for world in (1, 2, 3, 8):
            spans = [D.token_slice(m, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == m
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))


def _sharded_worker(rank, world, port, chunks, results):
    import torch
    import torch.distributed as dist

    from oracle import tilesparse_oracle as orc

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a, enc = _problem()
        # the per-rank product stands in for K1 (no GPU here): the oracle on
        # this rank's tile group, written into the shard view like K1 does
        lo, hi = D.column_shards(enc, world)[rank]
        sub = D.shard_encoding(enc, lo, hi)

        def local(x, out):
            out.copy_(torch.from_numpy(orc.c_gemm_cto_enc(x.t().numpy().copy(), sub).T))

        sp = D.TwShardedPlan(enc, chunks=chunks, local_product=local)
        at = torch.from_numpy(np.ascontiguousarray(a.T))
        res = sp.run(at, out_dtype="fp32")
        full = res.full() if isinstance(res, D.ChunkedRows) else res
        if isinstance(res, D.ChunkedRows):
            assert len(res.parts) == len(D.token_chunks(a.shape[0], chunks))
        results[rank] = (full.numpy().T.copy(), sp.condensed_columns.copy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,chunks", [(2, 1), (2, 3), (3, 2)])
def test_sharded_plan_all_gathers_full_product(world, chunks):
    """TwShardedPlan: every rank ends with the whole condensed product (the
    column shards all-gathered, M-chunked when chunks > 1) equal to the
    single-device product, with the reference's condensed column map."""
    from oracle import tilesparse_oracle as orc

    a, enc = _problem()
    want = orc.c_gemm_cto_enc(a, enc)
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_sharded_worker, args=(world, _free_port(), chunks, results), nprocs=world,
             join=True)
    kept = np.concatenate([np.arange(int(enc.col_counts[i])) +
                           enc.col_offsets[i, :int(enc.col_counts[i])]
                           for i in range(enc.tile_count)])
    for r in range(world):
        got, cols = results[r]
        assert np.allclose(got, want, rtol=0, atol=1e-5 * np.abs(want).max())
        assert np.array_equal(cols, kept)


def test_split_sms_floors_and_total():
    b = tw.split_sms([10, 40, 35], [3, 12, 3], 148)
    assert sum(b) == 148 and b[1] >= 12 and all(x >= f for x, f in zip(b, [3, 12, 3]))
    assert tw.split_sms([1, 1], [70, 70], 148)[0] >= 70
    with pytest.raises(tw.InvalidInputError):
        tw.split_sms([1, 1], [100, 100], 148)


def test_tune_budgets_hill_climbs_to_measured_minimum():
    """tune_budgets (the measured refinement of TwPlanGroup's SM shares)
    walks coordinate moves from the model's shares to the fastest measured
    candidate, respecting every plan's sub-tile floor and the SM total."""
    from types import SimpleNamespace

    from paper_2402_10876_b200.group import tune_budgets

    class FakeGroup:
        def __init__(self, budgets, floors):
            self.budgets = list(budgets)
            self.plans = [SimpleNamespace(info=SimpleNamespace(n_sub=f)) for f in floors]

        def set_budgets(self, b):
            assert all(x >= p.info.n_sub for x, p in zip(b, self.plans))
            assert sum(b) <= 148
            self.budgets = list(b)

    groups = [FakeGroup([16, 84, 48], [3, 12, 3]) for _ in range(2)]
    target = (22, 80, 46)

    def time_fn():
        b = groups[0].budgets
        assert groups[1].budgets == b          # every group moves together
        return sum(abs(x - t) for x, t in zip(b, target)) + 10.0

    best, t, seen = tune_budgets(groups, time_fn, moves=(4, 2), rounds=4)
    assert tuple(best) == target and t == 10.0
    assert groups[0].budgets == best and all(sum(k) == 148 for k in seen)
