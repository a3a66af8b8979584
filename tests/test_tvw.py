"""TVW (tile-wise + fixed 2:4 down every payload column, reference
patterns.py:645-717): the host restatement against the reference's own
outputs (tests/golden/tvw.npz, made by tests/golden/make_golden_tvw.py), the
oracle on TVW payloads, and -- on the GPU -- the product through K1."""

from __future__ import annotations

import json

import numpy as np
import pytest

from helpers import golden_str, load_npz, sha

import paper_2402_10876_b200 as tw
from oracle import tilesparse_oracle as orc

TOL = {"fp32": 1e-5, "fp16": 1e-3}


def test_small_cases_bit_exact():
    z, meta = load_npz("tvw.npz")
    for i, m in enumerate(meta):
        p = f"c{i}_"
        plan, tsm, vw = tw.prune_tvw(z[p + "w"], m["s"], m["g"])
        assert np.array_equal(np.packbits(plan.element_mask.ravel()), z[p + "mask"]), i
        assert np.array_equal(tsm.column_mask.kept, z[p + "cols"]), i
        assert np.array_equal(np.concatenate([t.kept_rows.kept for t in tsm.tiles]), z[p + "rows"])
        payload = np.concatenate([t.payload.ravel() for t in tsm.tiles])
        assert payload.tobytes() == z[p + "payload"].tobytes(), i     # incl. signed zeros
        offs = np.concatenate([o.ravel() for o in vw.kept_offsets])
        assert offs.dtype == np.int8 and np.array_equal(offs, z[p + "offsets"]), i
        doc = json.loads(bytes(z[p + "params"]).decode())
        assert doc["params"] == json.loads(json.dumps(plan.params, sort_keys=True)), i
        assert doc["clamps"] == plan.clamps and doc["achieved"] == plan.achieved_sparsity, i
        # every complete 4-vector of every payload column keeps exactly 2
        for t in tsm.tiles:
            full = t.payload.shape[0] // 4 * 4
            nz = (t.payload[:full].reshape(-1, 4, t.payload.shape[1]) != 0).sum(axis=1)
            assert nz.max(initial=0) <= 2
        # the oracle reproduces the reference product on TVW payloads bit for bit
        out = orc.c_gemm_cto_enc(z[p + "a"], tw.encode_cto(tsm), threads=2)
        assert np.array_equal(out, z[p + "out"]), i


def test_bert_structure_and_oracle_bit_exact():
    z, _ = load_npz("tvw.npz")
    w = tw.round_to(tw.synthetic_matrix(0, 768, 768, tw.STREAM_WEIGHTS), "fp16")
    plan, tsm, vw = tw.prune_tvw(w, 0.75, 128)
    enc = tw.encode_cto(tsm)
    assert sha(plan.element_mask) == golden_str(z, "bert_mask_sha256")
    assert sha(enc.payload) == golden_str(z, "bert_payload_sha256")
    assert sha(np.concatenate([o.ravel() for o in vw.kept_offsets])) == golden_str(
        z, "bert_offsets_sha256")
    for key in ("row_offsets", "col_offsets", "row_counts", "col_counts"):
        assert np.array_equal(getattr(enc, key), z["bert_" + key]), key
    a = tw.round_to(tw.synthetic_matrix(0, 8192, 768, tw.STREAM_INPUT), "fp16")
    out = orc.c_gemm_cto_enc(a, enc, threads=4)
    assert sha(out) == golden_str(z, "bert_out_sha256")


def test_rejections_and_dispatch():
    w = np.arange(64, dtype=np.float32).reshape(8, 8)
    with pytest.raises(tw.InvalidInputError):
        tw.prune_tvw(w, 0.4, 4)                       # below the 2:4 floor
    res = tw.prune_matrix("tvw", w, 0.75, g=4)
    assert res.vw_meta is not None and res.vw_meta.keep_per_vector == 2
    assert res.plan.params["tw_share"] == 0.5
    assert abs(res.plan.achieved_sparsity - 0.75) <= res.plan.params["slack_bound"]


@pytest.mark.gpu
@pytest.mark.parametrize("layout", ["natural", "runs"])
def test_tvw_gemm_matches_golden_and_oracle(layout):
    z, _ = load_npz("tvw.npz")
    w = tw.round_to(tw.synthetic_matrix(0, 768, 768, tw.STREAM_WEIGHTS), "fp16")
    a = tw.round_to(tw.synthetic_matrix(0, 8192, 768, tw.STREAM_INPUT), "fp16")
    _, tsm, _ = tw.prune_tvw(w, 0.75, 128)
    enc = tw.encode_cto(tsm)
    plan = tw.TwPlan(enc, row_layout=layout)
    got = plan.run(plan.prepare(a)).t()
    assert tw.relative_error(got[:8].cpu().numpy(), z["bert_out8"]) <= TOL["fp32"]
    assert tw.relative_error(got, orc.c_gemm_cto_enc(a, enc, threads=8)) <= TOL["fp32"]
    out = tw.gemm_cto(a, enc, out_dtype="fp16")
    assert tw.relative_error(out.condensed.float(), got) <= TOL["fp16"]


@pytest.mark.gpu
@pytest.mark.parametrize("k,n,m,compute", [(768, 768, 8192, "fp16"), (768, 3072, 1000, "fp16"),
                                           (512, 384, 333, "bf16"), (1024, 1024, 128, "fp16")])
def test_tvw_sparse_tensor_cores_match_oracle(k, n, m, compute, monkeypatch):
    """TVW through tcgen05.mma.sp (TW_SPARSE=1): the compressed 2:4 payload
    and the TMEM metadata (layout pinned by scripts/sp_probe.cu) give the
    oracle's product; the dense tensor-core path on the same plan agrees."""
    monkeypatch.setenv("TW_SPARSE", "1")
    rng = np.random.default_rng(k + n + m)
    w = tw.round_to(rng.normal(size=(k, n)).astype(np.float32), compute)
    a = tw.round_to(rng.normal(size=(m, k)).astype(np.float32), compute)
    _, tsm, _ = tw.prune_tvw(w, 0.75, 128)
    enc = tw.encode_cto(tsm)
    plan = tw.TwPlan(enc, compute_dtype=compute)
    assert plan.info.sparse_payload == 1
    x = plan.prepare(a)
    got = plan.run(x).t()
    idx = np.arange(0, m, max(1, m // 512))
    ref = orc.c_gemm_cto_enc(a[idx], enc, threads=8)
    import torch
    sel = torch.as_tensor(idx, device=got.device)
    assert tw.relative_error(got[sel].cpu().numpy(), ref) <= TOL["fp32"]
    monkeypatch.setenv("TW_NO_SPARSE", "1")
    dense = plan.run(x).t()
    assert tw.relative_error(got, dense) <= TOL["fp32"]


@pytest.mark.gpu
def test_tvw_sparse_declines_non_24_payloads(monkeypatch):
    """A TW payload (no 2:4 structure) never takes the sparse path."""
    monkeypatch.setenv("TW_SPARSE", "1")
    rng = np.random.default_rng(3)
    w = tw.round_to(rng.normal(size=(256, 256)).astype(np.float32), "fp16")
    _, tsm = tw.prune_tw(w, 0.5, 128)
    plan = tw.TwPlan(tw.encode_cto(tsm))
    assert plan.info.sparse_payload == 0
