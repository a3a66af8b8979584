"""Host prune / compress (the product's host code) vs the reference's golden
vectors: masks, indices, offsets and overlays must be bit-exact."""

from __future__ import annotations

import math
from fractions import Fraction

import numpy as np
import pytest

from helpers import golden_str, load_npz, sha, tiles_from_record

import paper_2402_10876_b200 as tw


def _check_record(z, prefix, plan, tsm, full_mask=True):
    enc = tw.encode_cto(tsm)
    if full_mask:
        golden = np.unpackbits(z[prefix + "mask"])[:plan.element_mask.size]
        assert np.array_equal(plan.element_mask.ravel(), golden.astype(bool))
    assert sha(plan.element_mask) == golden_str(z, prefix + "mask_sha256")
    assert np.array_equal(tsm.column_mask.kept, z[prefix + "cols"])
    for t, rows in zip(tsm.tiles, tiles_from_record(z, prefix)):
        assert np.array_equal(t.kept_rows.kept, rows)
    for f in ("row_counts", "col_counts", "row_offsets", "col_offsets"):
        assert np.array_equal(getattr(enc, f), z[prefix + f]), f
    assert sha(enc.payload) == golden_str(z, prefix + "payload_sha256")


def test_small_cases_bit_exact():
    z, meta = load_npz("small.npz")
    for ci, m in enumerate(meta):
        p = f"c{ci}_"
        w = z[p + "w"]
        plan, tsm = tw.prune_tw(w, m["s"], m["g"])
        _check_record(z, p + "tw_", plan, tsm)
        assert plan.achieved_sparsity == m["tw_achieved"]
        assert plan.clamps == m["tw_clamps"]
        assert plan.params == m["tw_params"]
        if m["tew"]:
            tplan, ttsm, ov = tw.prune_tew(w, m["s"], m["delta"], m["g"])
            _check_record(z, p + "tew_", tplan, ttsm)
            assert np.array_equal(ov.col_ptr, z[p + "tew_col_ptr"])
            assert np.array_equal(ov.row_idx, z[p + "tew_row_idx"])
            assert ov.values.tobytes() == z[p + "tew_values"].tobytes()
            assert tplan.achieved_sparsity == m["tew_achieved"]
            assert tplan.params == m["tew_params"]


def test_bert_structure_bit_exact():
    z, meta = load_npz("bert.npz")
    for li, info in enumerate(meta):
        k, n = info["k"], info["n"]
        w = tw.round_to(tw.synthetic_matrix(0, k, n, tw.STREAM_WEIGHTS), "fp16")
        plan, tsm = tw.prune_tw(w, 0.75, 128)
        _check_record(z, f"l{li}_tw_", plan, tsm, full_mask=False)
        assert plan.achieved_sparsity == info["tw_achieved"]
        tplan, ttsm, ov = tw.prune_tew(w, 0.75, 0.015, 128)
        _check_record(z, f"l{li}_tew_", tplan, ttsm, full_mask=False)
        assert ov.nnz == info["tew_nnz"]
        assert np.array_equal(ov.col_ptr, z[f"l{li}_tew_col_ptr"])
        assert np.array_equal(ov.row_idx, z[f"l{li}_tew_row_idx"])
        assert ov.values.tobytes() == z[f"l{li}_tew_values"].tobytes()
        assert tplan.clamps == info["tew_clamps"]


def test_cfg1_structure():
    z, meta = load_npz("cfg1.npz")
    w = tw.synthetic_matrix(0, 1024, 1024, tw.STREAM_WEIGHTS)
    plan, tsm = tw.prune_tw(w, 0.75, 128)
    _check_record(z, "tw_", plan, tsm, full_mask=False)
    assert tw.report(plan, tsm, 128).sparse_flops == meta["flops"]


# ---- known answers from the reference's own tests ---------------------------

def test_floor_count_exact():                      # test_core.py:56-61
    assert tw.floor_count(0.37, 100) == 37
    assert tw.floor_count(0.5, 7) == 3
    assert tw.floor_count(0.0, 10) == 0
    for s in (0.1, 0.3, 0.75, 0.9, 0.95):
        for n in (7, 100, 768, 12345):
            exact = math.floor(Fraction(s) * n)
            assert tw.floor_count(s, n) in (exact, exact + 1)


def test_split_is_half_half():                     # test_acceptance.py:119-135
    rng = np.random.default_rng(0)
    plan, _ = tw.prune_tw(rng.normal(size=(64, 64)).astype(np.float32), 0.75, 8)
    assert plan.params["column_share"] == 0.5 and plan.params["row_share"] == 0.5


def test_zero_sparsity_widths():                   # test_patterns.py:153-159
    rng = np.random.default_rng(1)
    _, tsm = tw.prune_tw(rng.normal(size=(6, 10)).astype(np.float32), 0.0, 4)
    assert tsm.tile_widths == [4, 4, 2]


def test_two_tile_worked_example():                # test_executor.py:140-154
    rng = np.random.default_rng(8)
    w = rng.normal(size=(5, 4)).astype(np.float32)
    mask = np.zeros((5, 4), dtype=bool)
    mask[[1, 2, 4], 0:2] = True
    mask[[0, 3], 2:4] = True
    enc = tw.encode_cto(tw.to_tile_sparse(w, mask, tw.TileConfig(granularity_g=2)))
    assert enc.row_offsets[0].tolist() == [1, 1, 2]
    assert enc.row_offsets[1].tolist() == [0, 2, 0]
    assert enc.row_counts.tolist() == [3, 2]


def test_all_kept_offsets():                       # test_formats.py:64-72
    w = np.arange(12, dtype=np.float32).reshape(3, 4) + 1
    enc = tw.encode_cto(tw.prune_tw(w, 0.0, 4)[1])
    assert enc.row_offsets[0].tolist() == [0, 0, 0]


def test_clamp_rows_unmet():                       # test_patterns.py:236-248
    w = np.ones((4, 8), dtype=np.float32)
    w[:, :4] = 10.0
    plan, tsm = tw.prune_tw(w, 0.9, 4)
    assert all(t.kept_rows.n_kept >= 1 for t in tsm.tiles)


def test_tew_cardinality():                        # test_patterns.py:264-280
    rng = np.random.default_rng(3)
    w = rng.normal(size=(16, 16)).astype(np.float32)
    plan, tsm, ov = tw.prune_tew(w, 0.5, 0.1, 4)
    assert ov.nnz == tw.floor_count(0.1, 256)
    assert not np.any(tsm.keep_mask() & (ov.to_dense() != 0))


def test_cto_round_trip_and_file(tmp_path):        # test_formats.py:82-98, 162-230
    rng = np.random.default_rng(4)
    for trial in range(20):
        k, n = int(rng.integers(1, 40)), int(rng.integers(1, 40))
        w = rng.normal(size=(k, n)).astype(np.float32)
        _, tsm = tw.prune_tw(w, float(rng.choice([0.0, 0.5, 0.8])), int(rng.integers(1, 9)))
        enc = tw.encode_cto(tsm)
        back = tw.decode_cto(enc)
        assert np.array_equal(back.reconstruct(), tsm.reconstruct())
        path = tmp_path / f"t{trial}.cto1"
        tw.write_cto1(path, enc)
        got = tw.read_cto1(path)
        assert got.payload.tobytes() == enc.payload.tobytes()
        assert np.array_equal(got.row_offsets, enc.row_offsets)
    data = bytearray(path.read_bytes())
    with pytest.raises(tw.CorruptEncodingError):
        (tmp_path / "trunc.cto1").write_bytes(bytes(data[:-3]))
        tw.read_cto1(tmp_path / "trunc.cto1")
    data[0:4] = b"XXXX"
    (tmp_path / "bad.cto1").write_bytes(bytes(data))
    with pytest.raises(tw.CorruptEncodingError):
        tw.read_cto1(tmp_path / "bad.cto1")


def test_corrupt_offsets_decode():                 # test_formats.py:112-159
    rng = np.random.default_rng(5)
    _, tsm = tw.prune_tw(rng.normal(size=(12, 8)).astype(np.float32), 0.6, 4)
    enc = tw.encode_cto(tsm)
    rows = enc.row_offsets.copy()
    rows[0, 0] = 5000
    bad = tw.CtoEncoding(original_dims=enc.original_dims, config=enc.config,
                         row_counts=enc.row_counts, col_counts=enc.col_counts, row_offsets=rows,
                         col_offsets=enc.col_offsets, payload=enc.payload)
    with pytest.raises(tw.CorruptEncodingError):
        tw.decode_cto(bad)
    with pytest.raises(tw.CorruptEncodingError):
        tw.CtoEncoding(original_dims=enc.original_dims, config=enc.config,
                       row_counts=enc.row_counts, col_counts=enc.col_counts,
                       row_offsets=enc.row_offsets, col_offsets=enc.col_offsets,
                       payload=enc.payload[:-1])


def test_rejections():
    with pytest.raises(tw.InvalidInputError):
        tw.prune_tw(np.ones((2, 2), np.float32), 1.0, 2)
    with pytest.raises(tw.InvalidInputError):
        tw.prune_tew(np.ones((2, 2), np.float32), 0.9, 0.2, 2)
    with pytest.raises(tw.InvalidInputError):
        tw.prune_tw(np.array([[np.inf, 1.0]], np.float32), 0.5, 1)
    with pytest.raises(tw.InvalidInputError):
        tw.prune_matrix("ew", np.ones((2, 2), np.float32), 0.5)
    with pytest.raises(tw.InvalidInputError):
        tw.as_matrix(np.ones(3))


def test_schedule_tiles_known_answers():           # test_executor.py:325-337
    assert tw.schedule_tiles([1, 1, 1, 1, 1], 2, "round_robin") == [0, 1, 0, 1, 0]
    a = tw.schedule_tiles([100, 10, 10, 10], 2, "lpt")
    assert all(x != a[0] for x in a[1:])
    with pytest.raises(tw.InvalidInputError):
        tw.schedule_tiles([1], 1, "random")
    with pytest.raises(tw.InvalidInputError):
        tw.schedule_tiles([1], 0)


def test_report_flops():                           # test_metrics.py:35-61
    rng = np.random.default_rng(6)
    w = rng.normal(size=(32, 48)).astype(np.float32)
    plan, tsm, ov = tw.prune_tew(w, 0.5, 0.05, 8)
    rep = tw.report(plan, tsm, 10, overlay=ov)
    assert rep.sparse_flops == 2 * 10 * (sum(t.width * t.kept_rows.n_kept for t in tsm.tiles)
                                         + ov.nnz)
    assert rep.dense_flops == 2 * 10 * 32 * 48


def test_relative_error_conventions():             # test_executor.py:385-390
    z = np.zeros((2, 2))
    assert tw.relative_error(z, z) == 0.0
    assert tw.relative_error(np.ones((2, 2)), z) == np.inf


def _big_fingerprint(plan, tsm, enc, ov=None):
    import hashlib

    def sha(a):
        return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()

    d = {"mask": sha(plan.element_mask),
         "cols": sha(np.asarray(tsm.column_mask.kept).astype(np.int64)),
         "rows": sha(np.concatenate([t.kept_rows.kept for t in tsm.tiles]).astype(np.int64)),
         "row_counts": enc.row_counts.astype(int).tolist(),
         "col_counts": enc.col_counts.astype(int).tolist(),
         "row_offsets": sha(enc.row_offsets), "col_offsets": sha(enc.col_offsets),
         "payload": sha(enc.payload), "achieved": float(plan.achieved_sparsity)}
    if ov is not None:
        d.update({"ov_col_ptr": sha(np.asarray(ov.col_ptr).astype(np.int64)),
                  "ov_row_idx": sha(np.asarray(ov.row_idx).astype(np.int64)),
                  "ov_values": sha(np.asarray(ov.values).astype(np.float32)),
                  "ov_nnz": int(ov.nnz)})
    return d


def _big_golden():
    import json
    from pathlib import Path

    return json.loads((Path(__file__).parent / "golden" / "big.json").read_text())


def test_prune_tw_bit_exact_at_16384():
    """configs[4]'s 16384 x 16384 weight: masks, kept columns, every tile's
    kept rows, CTO offsets and payload equal the reference's
    (tests/golden/make_golden_big.py fingerprints)."""
    want = _big_golden()["big_tw"]
    w = tw.round_to(tw.synthetic_matrix(0, 16384, 16384, tw.STREAM_WEIGHTS), "fp16")
    plan, tsm = tw.prune_tw(w, 0.75, 128)
    del w
    assert _big_fingerprint(plan, tsm, tw.encode_cto(tsm)) == want


def test_prune_tew_bit_exact_at_4096():
    want = _big_golden()["tew_4096"]
    w = tw.round_to(tw.synthetic_matrix(0, 4096, 4096, tw.STREAM_WEIGHTS), "fp16")
    plan, tsm, ov = tw.prune_tew(w, 0.75, 0.015, 128)
    assert _big_fingerprint(plan, tsm, tw.encode_cto(tsm), ov) == want


def test_prune_tw_bit_exact_vgg_sweep_shapes():
    """configs[3] VGG-16 im2col weights over the sparsity / G sweep."""
    gold = _big_golden()
    shapes = {"conv1_2": (576, 64), "conv2_1": (576, 128), "conv3_2": (2304, 256),
              "conv4_2": (4608, 512), "conv5_1": (4608, 512)}
    for name, (k, n) in shapes.items():
        w = tw.round_to(tw.synthetic_matrix(0, k, n, tw.STREAM_WEIGHTS), "fp16")
        for s in (0.5, 0.7, 0.9):
            for g in (64, 128, 256):
                plan, tsm = tw.prune_tw(w, s, g)
                got = _big_fingerprint(plan, tsm, tw.encode_cto(tsm))
                assert got == gold[f"{name}_s{s}_g{g}"], (name, s, g)
