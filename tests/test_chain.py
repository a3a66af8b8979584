"""Layer chaining in the condensed C'^T layout and CTO1 ->
device plans (8f-2).

CPU: the chained encoding of layer l+1 applied to layer l's condensed output
equals layer l+1 applied to the expanded output (zeros at pruned columns),
exactly (the oracle sums in fp64 in ascending row order; the dropped terms are
products with exact zeros).  GPU: the chained plan consumes layer l's C'^T
buffer directly.
"""

from __future__ import annotations

import numpy as np
import pytest

import paper_2402_10876_b200 as tw
from oracle import tilesparse_oracle as orc


def _layers(seed=0, k=256, n1=512, n2=192, s1=0.75, s2=0.6, g=64):
    rng = np.random.default_rng(seed)
    w1 = tw.round_to(rng.normal(size=(k, n1)).astype(np.float32), "fp16")
    w2 = tw.round_to(rng.normal(size=(n1, n2)).astype(np.float32), "fp16")
    _, t1 = tw.prune_tw(w1, s1, g)
    _, t2 = tw.prune_tw(w2, s2, g)
    return tw.encode_cto(t1), t1, tw.encode_cto(t2), t2


def test_chain_encoding_equals_expanded_product():
    e1, t1, e2, t2 = _layers()
    rng = np.random.default_rng(1)
    a = tw.round_to(rng.normal(size=(40, 256)).astype(np.float32), "fp16")
    h = orc.c_gemm_cto_enc(a, e1).astype(np.float32)          # condensed M x N1'
    full = np.zeros((h.shape[0], e2.original_dims[0]), dtype=np.float32)
    full[:, t1.column_mask.kept] = h                           # GemmOutput.expand
    ref = orc.c_gemm_cto_enc(full, e2)
    chained = tw.chain_encoding(e2, t1.column_mask.kept)
    assert chained.original_dims == (t1.n_condensed, e2.original_dims[1])
    out = orc.c_gemm_cto_enc(h, chained)
    assert np.array_equal(out, ref)
    # only MACs on surviving inputs remain
    assert int(chained.row_counts.sum()) <= int(e2.row_counts.sum())


def test_chain_tile_with_no_surviving_rows_outputs_zero():
    rng = np.random.default_rng(3)
    w2 = tw.round_to(rng.normal(size=(64, 16)).astype(np.float32), "fp16")
    _, t2 = tw.prune_tw(w2, 0.5, 8)
    e2 = tw.encode_cto(t2)
    # previous layer kept only rows no tile of layer 2 uses
    used = set()
    for i in range(e2.tile_count):
        used.update(e2.tile_rows(i).tolist())
    unused = [r for r in range(64) if r not in used]
    prev = unused if unused else [0]
    chained = tw.chain_encoding(e2, prev)
    h = rng.normal(size=(5, len(prev))).astype(np.float32)
    out = orc.c_gemm_cto_enc(h, chained)
    full = np.zeros((5, 64), dtype=np.float32)
    full[:, prev] = h
    assert np.array_equal(out, orc.c_gemm_cto_enc(full, e2))


def test_chain_rejects_bad_columns():
    _, _, e2, _ = _layers()
    with pytest.raises(tw.InvalidInputError):
        tw.chain_encoding(e2, [3, 2])
    with pytest.raises(tw.InvalidInputError):
        tw.chain_encoding(e2, [0, e2.original_dims[0]])


@pytest.mark.gpu
def test_chained_plans_on_gpu():
    """layer 1 -> C'^T (fp16) -> chained layer 2 reads it in place."""
    import torch

    e1, t1, e2, t2 = _layers(seed=5, k=768, n1=3072, n2=768, s1=0.75, s2=0.75, g=128)
    rng = np.random.default_rng(6)
    a = tw.round_to(rng.normal(size=(1000, 768)).astype(np.float32), "fp16")
    p1 = tw.TwPlan(e1)
    p2 = tw.TwPlan(tw.chain_encoding(e2, p1.condensed_columns))
    h = p1.run(p1.prepare(a), out_dtype="fp16")               # N1' x M, the next A^T
    out = p2.run(h)                                             # no expand / transpose
    hh = h.t().float().cpu().numpy()
    full = np.zeros((1000, 3072), dtype=np.float32)
    full[:, t1.column_mask.kept] = hh
    ref = orc.c_gemm_cto_enc(full, e2)
    assert tw.relative_error(out.t(), ref) <= 1e-5
    torch.cuda.synchronize()


@pytest.mark.gpu
def test_plan_from_cto1_file(tmp_path):
    e1, t1, _, _ = _layers(seed=7)
    path = tmp_path / "w.cto1"
    tw.write_cto1(path, e1)
    a = tw.round_to(np.random.default_rng(8).normal(size=(64, 256)).astype(np.float32), "fp16")
    p = tw.TwPlan.from_cto1(path)
    out = p.run(p.prepare(a))
    assert tw.relative_error(out.t(), orc.c_gemm_cto_enc(a, e1)) <= 1e-5


@pytest.mark.gpu
@pytest.mark.parametrize("m,splitk", [(1000, None), (64, "1")])
def test_chain_plans_write_next_layers_run_layout(m, splitk, monkeypatch):
    """chain_plans (BERT FFN shapes): layer l's epilogue writes C'^T directly
    in layer l+1's row-run order (payload rows permuted inside sub-tiles), and
    layer l+1 reads it with dense TMA boxes -- no prepare pass in between.
    Both products match the oracle on the same (fp16-rounded) values.  At
    m = 64 with TW_SPLITK=1 both layers run split-K (splitk_reduce writes
    the permuted order)."""
    import torch

    if splitk:
        monkeypatch.setenv("TW_SPLITK", splitk)
    rng = np.random.default_rng(5)
    w1 = tw.round_to(rng.normal(size=(768, 3072)).astype(np.float32), "fp16")
    w2 = tw.round_to(rng.normal(size=(3072, 768)).astype(np.float32), "fp16")
    _, t1 = tw.prune_tw(w1, 0.75, 128)
    _, t2 = tw.prune_tw(w2, 0.75, 128)
    e1, e2 = tw.encode_cto(t1), tw.encode_cto(t2)
    prev, nxt = tw.chain_plans(e1, e2)
    assert nxt.uses_row_runs
    # prev's output rows are a permutation of the condensed columns, inside
    # each 128-row sub-tile block
    cols = prev.condensed_columns
    assert sorted(cols.tolist()) == sorted(t1.column_mask.kept.tolist())
    b = prev.output_groups()
    kept = np.asarray(t1.column_mask.kept)
    for lo, hi in zip(b[:-1], b[1:]):
        assert sorted(cols[lo:hi].tolist()) == kept[lo:hi].tolist()
    a = tw.round_to(rng.normal(size=(m, 768)).astype(np.float32), "fp16")
    h = prev.run(prev.prepare(a), out_dtype="fp16")             # N1' x M, next's layout
    ref1 = orc.c_gemm_cto_enc(a, e1)                            # M x N1', condensed order
    pos = {int(c): i for i, c in enumerate(kept)}
    perm = np.array([pos[int(c)] for c in cols])
    assert tw.relative_error(h.float().t().cpu().numpy(), ref1[:, perm]) <= 1e-3
    y = nxt.run(h)                                              # TMA runs on h in place
    hn = h.float().t().cpu().numpy()                            # the values layer 2 read
    full = np.zeros((a.shape[0], 3072), dtype=np.float32)
    full[:, cols] = hn
    ref2 = orc.c_gemm_cto_enc(full, e2)
    assert tw.relative_error(y.t(), ref2) <= 1e-5
    # the same chain through the natural layouts gives the same numbers
    y_nat = tw.TwPlan(tw.chain_encoding(e2, kept)).run(
        tw.TwPlan(e1).run(tw.prepare_activations(a), out_dtype="fp16"))
    assert tw.relative_error(y.t(), y_nat.t().cpu().numpy()) <= 1e-5


@pytest.mark.gpu
@pytest.mark.parametrize("layout,overlay", [("runs", False), ("natural", False), ("runs", True)])
def test_device_plan_file_round_trip(tmp_path, layout, overlay):
    """TwPlan.save / TwPlan.load ("TWP1", the cached device-native format):
    the loaded plan computes bit-identical products (TW, and TEW with the
    overlay attached after loading); a corrupted file raises."""
    import torch

    rng = np.random.default_rng(9)
    w = tw.round_to(rng.normal(size=(768, 3072)).astype(np.float32), "fp16")
    a = tw.round_to(rng.normal(size=(700, 768)).astype(np.float32), "fp16")
    if overlay:
        _, tsm, ov = tw.prune_tew(w, 0.75, 0.015, 128)
    else:
        _, tsm = tw.prune_tw(w, 0.75, 128)
        ov = None
    enc = tw.encode_cto(tsm)
    p1 = tw.TwPlan(enc, row_layout=layout)
    n = p1.save(tmp_path / "plan.twp")
    assert n > 0
    p2 = tw.TwPlan.load(tmp_path / "plan.twp", overlay=ov)
    if ov is not None:
        p1.attach_overlay(ov)
    assert np.array_equal(p1.condensed_columns, p2.condensed_columns)
    assert np.array_equal(p1.row_order, p2.row_order)
    x = p1.prepare(a)
    if ov is None:
        assert torch.equal(p1.run(x), p2.run(x))
    else:
        assert torch.equal(p1.run_tew(x), p2.run_tew(x))
        assert np.array_equal(p1.union_columns, p2.union_columns)
    raw = bytearray((tmp_path / "plan.twp").read_bytes())
    (tmp_path / "bad.twp").write_bytes(bytes(raw[: len(raw) // 2]))
    with pytest.raises(tw.CorruptEncodingError):
        tw.TwPlan.load(tmp_path / "bad.twp")
    raw[0] ^= 0xFF
    (tmp_path / "bad2.twp").write_bytes(bytes(raw))
    with pytest.raises(tw.CorruptEncodingError):
        tw.TwPlan.load(tmp_path / "bad2.twp")
