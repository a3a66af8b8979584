"""Pin the CPU oracle (oracle/) to the reference's own outputs.

The golden vectors in tests/golden were produced by importing the unmodified
reference (tests/golden/make_golden.py).  The C oracle must reproduce the
reference's fp64 gemm_cto output BIT-EXACTLY (same products, same ascending
kept-row order), checked by array equality on the small cases and by sha256
of the full-size outputs (config 1 at M=128, BERT layers at M=8192).
"""

from __future__ import annotations

import numpy as np
import pytest

from helpers import golden_str, load_npz, sha, tiles_from_record

import paper_2402_10876_b200 as tw
from oracle import tilesparse_oracle as orc


def _enc_from_record(z, prefix, k, n, g, payload):
    return tw.CtoEncoding(original_dims=(k, n), config=tw.TileConfig(g),
                          row_counts=z[prefix + "row_counts"], col_counts=z[prefix + "col_counts"],
                          row_offsets=z[prefix + "row_offsets"],
                          col_offsets=z[prefix + "col_offsets"], payload=payload)


def _payload(w, z, prefix):
    """Packed transposed payload rebuilt from the weights + golden structure."""
    cols = z[prefix + "cols"].astype(np.int64)
    rows = tiles_from_record(z, prefix)
    widths = z[prefix + "col_counts"].astype(np.int64)
    parts, pos = [], 0
    for r, wd in zip(rows, widths):
        parts.append(np.ascontiguousarray(w[np.ix_(r, cols[pos:pos + wd])].T).ravel())
        pos += wd
    return np.concatenate(parts).astype(np.float32)


def test_small_tw_bit_exact():
    z, meta = load_npz("small.npz")
    for ci, m in enumerate(meta):
        p = f"c{ci}_"
        w, a = z[p + "w"], z[p + "a"]
        payload = _payload(w, z, p + "tw_")
        assert sha(payload) == golden_str(z, p + "tw_payload_sha256")
        enc = _enc_from_record(z, p + "tw_", m["k"], m["n"], m["g"], payload)
        out = orc.c_gemm_cto_enc(a, enc, threads=2)
        assert np.array_equal(out, z[p + "tw_out"]), ci
        # the faithful numpy port of execute_batched agrees bit for bit too
        tiles = [(r, np.ascontiguousarray(w[np.ix_(r, c)]))
                 for r, c in zip(tiles_from_record(z, p + "tw_"),
                                 np.split(z[p + "tw_cols"].astype(np.int64),
                                          np.cumsum(z[p + "tw_col_counts"])[:-1]))]
        port = orc.execute_batched(a, tiles, workers=2)
        assert np.array_equal(port, z[p + "tw_out"]), ci


def test_small_tew_within_reference_tolerance():
    """gemm_tew sums the overlay with BLAS (executor.py:200, order unfixed);
    the reference's own tolerance for it is 1e-12 (test_executor.py:211-217)."""
    z, meta = load_npz("small.npz")
    seen = 0
    for ci, m in enumerate(meta):
        if not m["tew"]:
            continue
        p = f"c{ci}_"
        w, a = z[p + "w"], z[p + "a"]
        enc = _enc_from_record(z, p + "tew_", m["k"], m["n"], m["g"], _payload(w, z, p + "tew_"))
        out, union = orc.tew_reference(a, enc, z[p + "tew_col_ptr"], z[p + "tew_row_idx"],
                                       z[p + "tew_values"], m["n"])
        assert np.array_equal(union, z[p + "tew_union"])
        assert tw.relative_error(out, z[p + "tew_out"]) <= 1e-12
        seen += 1
    assert seen >= 10


def test_naive_prune_matches_golden_masks():
    """Plain-loop TW restatement == reference masks on tie-free cases."""
    z, meta = load_npz("small.npz")
    checked = 0
    for ci, m in enumerate(meta):
        p = f"c{ci}_"
        w = z[p + "w"]
        if m["k"] * m["n"] > 20000 or np.unique(np.abs(w)).size != w.size:
            continue
        mask, cols, rows = orc.naive_prune_tw(w, m["s"], m["g"])
        golden = np.unpackbits(z[p + "tw_mask"])[:w.size].reshape(w.shape).astype(bool)
        assert np.array_equal(mask, golden), ci
        assert np.array_equal(cols, z[p + "tw_cols"])
        if m["tew"]:
            restored = orc.naive_tew_restore(w, golden, m["delta"])
            tew_mask = np.unpackbits(z[p + "tew_mask"])[:w.size].reshape(w.shape).astype(bool)
            tw_mask2, _, _ = orc.naive_prune_tw(w, m["s"] + m["delta"], m["g"])
            flat = tw_mask2.ravel().copy()
            restored = orc.naive_tew_restore(w, tw_mask2, m["delta"])
            flat[restored] = True
            assert np.array_equal(flat.reshape(w.shape), tew_mask), ci
        checked += 1
    assert checked >= 15


def test_cfg1_full_output_sha():
    z, meta = load_npz("cfg1.npz")
    w = tw.synthetic_matrix(0, 1024, 1024, tw.STREAM_WEIGHTS)
    a = tw.synthetic_matrix(0, 128, 1024, tw.STREAM_INPUT)
    payload = _payload(w, z, "tw_")
    enc = _enc_from_record(z, "tw_", 1024, 1024, 128, payload)
    out = orc.c_gemm_cto_enc(a, enc)
    assert np.array_equal(out[:16], z["out16"])
    assert sha(out) == meta["out_sha256"]


@pytest.mark.slow
def test_bert_full_output_sha():
    """C oracle == reference at full BERT size (M=8192), by sha256 of the bytes."""
    z, meta = load_npz("bert.npz")
    for li, info in enumerate(meta):
        k, n = info["k"], info["n"]
        w = tw.round_to(tw.synthetic_matrix(0, k, n, tw.STREAM_WEIGHTS), "fp16")
        a = tw.round_to(tw.synthetic_matrix(0, 8192, k, tw.STREAM_INPUT), "fp16")
        p = f"l{li}_tw_"
        enc = _enc_from_record(z, p, k, n, 128, _payload(w, z, p))
        out = orc.c_gemm_cto_enc(a, enc)
        assert np.array_equal(out[:8], z[f"l{li}_tw_out8"])
        assert sha(out) == info["tw_out_sha256"], li


def test_mac_kernel_port_known_answer():
    """Rank-1 known answer of test_executor.py:92-99."""
    a = np.array([[1.0, 2.0], [3.0, 4.0]])
    out = orc.tile_product(a, np.array([0]), np.array([[5.0, 6.0]]))
    assert np.array_equal(out, [[5.0, 6.0], [15.0, 18.0]])


def test_schedule_port_known_answers():
    assert orc.schedule_tiles([1, 1, 1, 1, 1], 2, "round_robin") == [0, 1, 0, 1, 0]
    a = orc.schedule_tiles([100, 10, 10, 10], 2, "lpt")
    assert all(x != a[0] for x in a[1:])
