"""GPU parity: the sm_100a kernels (through the C ABI) vs the CPU oracle.

Protocol: inputs are rounded once to the compute
dtype; the oracle (fp64, reference accumulation order) and the GPU (fp32
TMEM accumulation) see identical values, so the only differences are fp32
accumulation order and output rounding.  Tolerances on
``relative_error`` (executor.py:278-288, max|diff| / max|ref|):

    fp32 out: 1e-5     fp16 out: 1e-3     bf16 out: 8e-3
"""

from __future__ import annotations

import numpy as np
import pytest

from helpers import load_npz, tiles_from_record

import paper_2402_10876_b200 as tw
from oracle import tilesparse_oracle as orc

pytestmark = pytest.mark.gpu

TOL = {"fp32": 1e-5, "fp16": 1e-3, "bf16": 8e-3}


def _rounded(x, dt="fp16"):
    return tw.round_to(x, dt)


def _problem(k, n, m, s, g, seed, dt="fp16"):
    rng = np.random.default_rng(seed)
    w = _rounded(rng.normal(size=(k, n)).astype(np.float32), dt)
    a = _rounded(rng.normal(size=(m, k)).astype(np.float32), dt)
    plan, tsm = tw.prune_tw(w, s, g)
    return w, a, plan, tsm


def _oracle_tw(a, tsm):
    return orc.c_gemm_cto_enc(a, tw.encode_cto(tsm))


@pytest.mark.parametrize("k,n,m,s,g", [
    (64, 64, 128, 0.5, 32),       # one 128-token block, single k-step
    (128, 256, 256, 0.75, 128),   # two tiles, two blocks
    (200, 150, 77, 0.6, 64),      # ragged M, ragged last tile
    (768, 768, 1000, 0.75, 128),  # BERT-shaped, M tail
    (96, 80, 5, 0.3, 16),         # M < 8 (padded pitch)
    (33, 17, 1, 0.5, 4),          # M = 1, tiny tiles
    (300, 700, 130, 0.5, 300),    # g > 256: tiles split into UMMA-N slices
    (50, 64, 64, 0.0, 8),         # nothing pruned
    (40, 400, 64, 0.9, 1),        # g = 1: 40 width-1 tiles
    # VGG-16 im2col shapes (configs[3]) at reduced M: K = 9 * C_in
    (27, 64, 4096, 0.5, 64),      # conv1_1: K = 27, one 64-wide tile
    (576, 128, 4096, 0.9, 256),   # conv2_1 at 90%: K' down to a few rows
    (2304, 512, 2048, 0.75, 128), # conv4_1
    (4608, 512, 1536, 0.9, 64),   # conv4_2 at 90%, G = 64
])
def test_tw_matches_oracle(k, n, m, s, g):
    w, a, plan, tsm = _problem(k, n, m, s, g, seed=k * 31 + n)
    out = tw.gemm_tile_sparse(a, tsm)
    ref = _oracle_tw(a, tsm)
    assert out.condensed.shape == ref.shape
    assert tw.relative_error(out.condensed, ref) <= TOL["fp32"]
    # expanded result vs masked dense: zeros at pruned columns
    full = out.expand().cpu().numpy()
    pruned = np.setdiff1d(np.arange(n), tsm.column_mask.kept)
    assert np.all(full[:, pruned] == 0)


def test_three_tw_paths_bit_identical():
    w, a, plan, tsm = _problem(256, 384, 300, 0.75, 128, seed=7)
    enc = tw.encode_cto(tsm)
    o1 = tw.gemm_tile_sparse(a, tsm).condensed
    o2 = tw.gemm_cto(a, enc, check_padding=True).condensed
    o3, trace = tw.execute_batched(a, tsm, workers=3)
    o4, _ = tw.execute_batched(a, tsm, workers=2, strategy="round_robin")
    for o in (o2, o3.condensed, o4.condensed):
        assert o.cpu().numpy().tobytes() == o1.cpu().numpy().tobytes()
    assert trace.total_macs == sum(300 * t.width * t.kept_rows.n_kept for t in tsm.tiles)


@pytest.mark.parametrize("out_dtype", ["fp32", "fp16", "bf16"])
@pytest.mark.parametrize("compute", ["fp16", "bf16"])
def test_dtypes(compute, out_dtype):
    w, a, plan, tsm = _problem(256, 256, 256, 0.75, 64, seed=3, dt=compute)
    out = tw.gemm_tile_sparse(a, tsm, compute_dtype=compute, out_dtype=out_dtype)
    ref = _oracle_tw(a, tsm)
    assert tw.relative_error(out.condensed, ref) <= TOL[out_dtype]


def test_bert_golden_rows():
    """First 8 tokens of every BERT layer vs the reference's own fp64 output."""
    z, meta = load_npz("bert.npz")
    for li, info in enumerate(meta):
        k, n = info["k"], info["n"]
        w = tw.round_to(tw.synthetic_matrix(0, k, n, tw.STREAM_WEIGHTS), "fp16")
        a = tw.round_to(tw.synthetic_matrix(0, 8192, k, tw.STREAM_INPUT), "fp16")
        plan, tsm = tw.prune_tw(w, 0.75, 128)
        rows = tiles_from_record(z, f"l{li}_tw_")
        assert all(np.array_equal(t.kept_rows.kept, r) for t, r in zip(tsm.tiles, rows))
        out = tw.gemm_cto(a, tw.encode_cto(tsm))
        got = out.condensed[:8].cpu().numpy()
        assert tw.relative_error(got, z[f"l{li}_tw_out8"]) <= TOL["fp32"]
        # full M = 8192 against the oracle (pinned to the reference by sha256)
        full = orc.c_gemm_cto_enc(a, tw.encode_cto(tsm))
        assert tw.relative_error(out.condensed, full) <= TOL["fp32"]


def test_tew_matches_oracle():
    rng = np.random.default_rng(11)
    k, n, m = 256, 320, 200
    w = _rounded(rng.normal(size=(k, n)).astype(np.float32))
    a = _rounded(rng.normal(size=(m, k)).astype(np.float32))
    plan, tsm, ov = tw.prune_tew(w, 0.6, 0.05, 64)
    out = tw.gemm_tew(a, tsm, ov)
    ref, union = orc.tew_reference(a, tw.encode_cto(tsm), ov.col_ptr, ov.row_idx, ov.values, n)
    assert np.array_equal(out.column_map.kept, union)
    assert tw.relative_error(out.condensed, ref) <= TOL["fp32"]
    # and against the masked dense fp64 product on the union mask
    dense = tw.masked_dense_reference(a, w, plan.element_mask)
    assert tw.relative_error(out.expand(), dense) <= TOL["fp32"]


@pytest.mark.parametrize("k,compute", [(4608, "fp16"), (4608, "bf16"), (3072, "bf16")])
def test_tew_block_sizes_match_oracle(k, compute):
    """K2 with the 16- and 32-token staged blocks (K > 1536 rows) and the
    bf16 kernel: every packed entry's block offset (row * T / 8) stays in 16
    bits up to the largest block, and the result matches the oracle."""
    rng = np.random.default_rng(k)
    n, m = 256, 203
    w = tw.round_to(rng.normal(size=(k, n)).astype(np.float32), compute)
    a = tw.round_to(rng.normal(size=(m, k)).astype(np.float32), compute)
    _, tsm, ov = tw.prune_tew(w, 0.75, 0.02, 128)
    out = tw.gemm_tew(a, tsm, ov, compute_dtype=compute)
    ref, union = orc.tew_reference(a, tw.encode_cto(tsm), ov.col_ptr, ov.row_idx, ov.values, n)
    assert np.array_equal(out.column_map.kept, union)
    assert tw.relative_error(out.condensed, ref) <= TOL["fp32"]


def test_tew_bert_golden_rows():
    z, meta = load_npz("bert.npz")
    for li, info in enumerate(meta):
        k, n = info["k"], info["n"]
        w = tw.round_to(tw.synthetic_matrix(0, k, n, tw.STREAM_WEIGHTS), "fp16")
        a = tw.round_to(tw.synthetic_matrix(0, 8192, k, tw.STREAM_INPUT), "fp16")
        plan, tsm, ov = tw.prune_tew(w, 0.75, 0.015, 128)
        assert ov.nnz == info["tew_nnz"]
        out = tw.gemm_tew(a, tsm, ov)
        assert np.array_equal(out.column_map.kept, z[f"l{li}_tew_union"])
        got = out.condensed[:8].cpu().numpy()
        assert tw.relative_error(got, z[f"l{li}_tew_out8"]) <= TOL["fp32"]


def test_empty_overlay_equals_tw():
    w, a, plan, tsm = _problem(64, 96, 40, 0.5, 32, seed=5)
    empty = tw.SparseOverlay.empty((64, 96))
    base = tw.gemm_tile_sparse(a, tsm).expand().cpu().numpy()
    out = tw.gemm_tew(a, tsm, empty).expand().cpu().numpy()
    assert np.array_equal(base, out)


def test_error_mapping():
    w, a, plan, tsm = _problem(48, 32, 16, 0.6, 8, seed=9)
    enc = tw.encode_cto(tsm)
    bad = enc.row_offsets.copy()
    bad[0, 0] = 5000
    corrupt = tw.CtoEncoding(original_dims=enc.original_dims, config=enc.config,
                             row_counts=enc.row_counts, col_counts=enc.col_counts,
                             row_offsets=bad, col_offsets=enc.col_offsets, payload=enc.payload)
    with pytest.raises(tw.CorruptEncodingError):
        tw.gemm_cto(a, corrupt)
    with pytest.raises(tw.InvalidInputError):
        tw.gemm_tile_sparse(np.ones((4, 47), np.float32), tsm)
    r, c = np.argwhere(tsm.keep_mask())[0]
    clash = tw.SparseOverlay.from_coords((48, 32), [r], [c], [1.0])
    with pytest.raises(tw.ContractViolationError):
        tw.gemm_tew(a, tsm, clash)
    with pytest.raises(tw.InvalidInputError):
        tw.gemm_tew(a, tsm, tw.SparseOverlay.empty((49, 32)))


def test_padding_never_dereferenced():
    """Corrupting only the padded region of the offsets leaves the result
    bit-identical (test_executor.py:156-180)."""
    w, a, plan, tsm = _problem(96, 64, 64, 0.6, 16, seed=13)
    enc = tw.encode_cto(tsm)
    clean = tw.gemm_cto(a, enc).condensed.cpu().numpy()
    rows = enc.row_offsets.copy()
    for i in range(enc.tile_count):
        rows[i, int(enc.row_counts[i]):] = 9999
    dirty = tw.CtoEncoding(original_dims=enc.original_dims, config=enc.config,
                           row_counts=enc.row_counts, col_counts=enc.col_counts,
                           row_offsets=rows, col_offsets=enc.col_offsets, payload=enc.payload)
    assert tw.gemm_cto(a, dirty).condensed.cpu().numpy().tobytes() == clean.tobytes()


def test_nonfinite_activation_not_in_padding():
    """A NaN in an activation row that no tile keeps must not leak into the
    output (gather padding is TMA out-of-bounds zero fill, not a real row)."""
    w, a, plan, tsm = _problem(64, 64, 128, 0.75, 32, seed=21)
    kept_any = np.zeros(64, bool)
    for t in tsm.tiles:
        kept_any[t.kept_rows.kept] = True
    dead = np.flatnonzero(~kept_any)
    if dead.size == 0:
        pytest.skip("every row kept by some tile")
    a2 = a.copy()
    a2[:, dead] = np.nan
    out = tw.gemm_tile_sparse(a2, tsm).condensed.cpu().numpy()
    assert np.all(np.isfinite(out))


@pytest.mark.parametrize("k,n,m,g,s", [
    (3072, 768, 8192, 128, 0.75),   # BERT FFN-2 shape: 192 units on 148 SMs -> stream-K
    (1000, 2000, 2500, 64, 0.6),    # ragged K' per tile, 20 blocks x 25 tiles
    (512, 4096, 4096, 256, 0.75),   # BN = 256
])
def test_stream_k_matches_oracle_and_is_deterministic(k, n, m, g, s):
    w, a, plan, tsm = _problem(k, n, m, s, g, seed=k + n + m)
    o1 = tw.gemm_tile_sparse(a, tsm).condensed.cpu().numpy()
    o2 = tw.gemm_tile_sparse(a, tsm).condensed.cpu().numpy()
    assert o1.tobytes() == o2.tobytes()
    assert tw.relative_error(o1, _oracle_tw(a, tsm)) <= TOL["fp32"]


@pytest.mark.parametrize("mode", ["owner", "strided"])
def test_streamed_modes_match_oracle(mode, monkeypatch):
    """K' > 448 (streamed payload) through both work decompositions."""
    monkeypatch.setenv("TW_OWNER" if mode == "owner" else "TW_STRIDED", "1")
    w, a, plan, tsm = _problem(2048, 1024, 1536, 0.75, 128, seed=7)
    out = tw.TwPlan(tw.encode_cto(tsm)).run(tw.prepare_activations(a)).t()
    assert tw.relative_error(out, _oracle_tw(a, tsm)) <= TOL["fp32"]


@pytest.mark.parametrize("world", [2, 3])
def test_column_shards_concatenate_bit_identical(world):
    """configs[4] partition on one GPU: every rank's shard plan writes its
    contiguous rows of C'^T; stacked in rank order they equal the unsharded
    product bit for bit (what the NCCL all-gather assembles)."""
    import torch

    from paper_2402_10876_b200 import distributed as D

    w, a, plan, tsm = _problem(1024, 2048, 1024, 0.75, 128, seed=world)
    enc = tw.encode_cto(tsm)
    full = tw.TwPlan(enc).run(tw.prepare_activations(a))
    shards = D.column_shards(enc, world)
    rows = D.shard_rows(enc, shards)
    parts = []
    for (lo, hi), (r0, r1) in zip(shards, rows):
        p = tw.TwPlan(D.shard_encoding(enc, lo, hi))
        part = p.run(p.prepare(a))
        assert part.shape[0] == r1 - r0
        parts.append(part)
    stacked = torch.cat(parts, dim=0)
    assert torch.equal(stacked, full)


@pytest.mark.parametrize("m,k,src,dst", [
    (8192, 768, "fp16", "fp16"),    # 16-byte tile path
    (136, 72, "bf16", "bf16"),      # 16-byte tile path, partial tiles
    (77, 50, "fp16", "fp16"),       # ragged: general path
    (64, 96, "fp32", "fp16"),       # cast: general path
    (40, 24, "fp32", "bf16"),
])
def test_transpose_cast_exact(m, k, src, dst):
    """K4 (A -> A^T + cast) equals torch's transpose + rounding bit for bit."""
    import torch

    dt = {"fp16": torch.float16, "bf16": torch.bfloat16, "fp32": torch.float32}
    g = torch.Generator(device="cuda").manual_seed(m + k)
    a = torch.randn((m, k), device="cuda", generator=g).to(dt[src])
    at = tw.prepare_activations(a, dst)
    assert tuple(at.shape) == (k, m)
    assert torch.equal(at, a.t().to(dt[dst]))


@pytest.mark.parametrize("k,n,m,s,g,env", [
    (768, 768, 1000, 0.75, 128, {}),                      # BERT 768^2 shape
    (3072, 768, 1000, 0.75, 128, {}),                     # BERT FFN-2 shape
    (3072, 768, 777, 0.75, 128, {"TW_STRIDED": "1"}),
    (768, 768, 600, 0.75, 128, {"TW_OWNER": "1"}),
    (768, 768, 1000, 0.75, 128, {"TW_RUN_MAX_UNITS": "0"}),  # plan layout via cp.async by position
    (4608, 512, 900, 0.9, 256, {}),                       # one wide tile (VGG conv4 shape)
    (1024, 512, 300, 0.5, 256, {}),                       # g = 256: 2 sub-tiles per tile
    (768, 3072, 1000, 0.75, 128, {"TW_RUN_COPIES": "3"}), # 12 tiles: one order per tile group
    (768, 3072, 8192, 0.75, 128, {"TW_RUN_COPIES": "3"}), # resident payload + runs, 3 units per CTA
    (768, 768, 16384, 0.75, 128, {}),                     # resident payload + runs, 4 units per CTA
])
def test_row_runs_layout_bit_identical(k, n, m, s, g, env, monkeypatch):
    """Plans with the row-run layout: activations prepared into the permuted
    row order and fetched with dense TMA boxes give exactly the result of the
    natural-order cp.async gather (same K' order), and match the oracle."""
    for name, value in env.items():
        monkeypatch.setenv(name, value)
    w, a, plan, tsm = _problem(k, n, m, s, g, seed=k + m)
    enc = tw.encode_cto(tsm)
    runs = tw.TwPlan(enc, row_layout="runs")
    assert runs.uses_row_runs, "expected a few-run row order for <= 6 tiles"
    copies = int(runs.info.row_copies)
    assert sorted(runs.row_order.tolist()) == sorted(list(range(k)) * copies)
    o_runs = runs.run(runs.prepare(a))                            # TMA row runs
    o_nat = runs.run(tw.prepare_activations(a), x_layout="natural")  # cp.async gather
    assert torch_equal(o_runs, o_nat)
    # natural A^T handed to a runs plan is permuted by prepare(at=...)
    o_at = runs.run(runs.prepare(at=tw.prepare_activations(a)))
    assert torch_equal(o_at, o_nat)
    assert tw.relative_error(o_runs.t(), _oracle_tw(a, tsm)) <= TOL["fp32"]


def torch_equal(x, y):
    import torch

    return torch.equal(x, y)


@pytest.mark.parametrize("out_dtype", ["fp32", "fp16"])
def test_tew_workspace_path_bit_identical(out_dtype):
    """TEW with the workspace (K1 -> condensed scratch, K2 scatters to union
    rows) equals the union-row scatter in K1 bit for bit."""
    import torch

    from paper_2402_10876_b200 import _native

    rng = np.random.default_rng(11)
    w = tw.round_to(rng.normal(size=(768, 768)).astype(np.float32), "fp16")
    a = tw.round_to(rng.normal(size=(700, 768)).astype(np.float32), "fp16")
    _, tsm, ov = tw.prune_tew(w, 0.75, 0.015, 128)
    plan = tw.TwPlan(tw.encode_cto(tsm), ov)
    x = plan.prepare(a)
    o_ws = plan.run_tew(x, out_dtype=out_dtype)
    o_sc = torch.empty_like(o_ws)
    lib = _native.load_library()
    _native.check(lib.tw_gemm_tew(plan._handle, x.data_ptr(), x.shape[1], x.stride(0),
                                  o_sc.data_ptr(), o_sc.stride(0),
                                  _native.TW_F32 if out_dtype == "fp32" else _native.TW_F16,
                                  _native.stream_handle()))
    assert torch.equal(o_ws, o_sc)


@pytest.mark.parametrize("sms,m", [(50, 8192), (24, 3001), (24, 8192)])
def test_paired_units_bit_identical(sms, m, monkeypatch):
    """TW_PAIR=1 (two units of a CTA's sub-tile share every streamed payload
    stage, accumulators 0 and 1) gives exactly the regular ring's output on a
    streamed row-run plan with several units per CTA, including a CTA with an
    odd unit count (its last unit runs alone)."""
    k, n = 3072, 768
    w = tw.round_to(tw.synthetic_matrix(0, k, n, tw.STREAM_WEIGHTS), "fp16")
    _, tsm = tw.prune_tw(w, 0.75, 128)
    plan = tw.TwPlan(tw.encode_cto(tsm), row_layout="runs")
    plan.set_sm_budget(sms)
    a = tw.round_to(tw.synthetic_matrix(0, m, k, tw.STREAM_INPUT), "fp16")
    x = plan.prepare(a)
    regular = plan.run(x, out_dtype="fp16")
    monkeypatch.setenv("TW_PAIR", "1")
    paired = plan.run(x, out_dtype="fp16")
    assert torch_equal(regular, paired)
    idx = np.arange(0, m, max(1, m // 64))
    ref = orc.c_gemm_cto_enc(a[idx], tw.encode_cto(tsm))
    assert tw.relative_error(paired.float().t().cpu().numpy()[idx], ref) <= TOL["fp16"]


@pytest.mark.parametrize("compute,m,out_dtype", [
    ("fp16", 8192, "fp16"), ("bf16", 4096, "bf16"), ("fp16", 1000, "fp16"), ("fp16", 640, "fp32"),
])
def test_tew_k2_16_tokens_per_lane_bit_identical(compute, m, out_dtype, monkeypatch):
    """K2 with 16 tokens per lane (the default for 64-token blocks) against
    the 8-token kernel (TW_K2_TPL=8 at plan creation): same entry order, same
    fp32 sums, so bit-identical outputs -- whole blocks (the 16-byte
    read-modify-write with the FHFMA add), a ragged last block and fp32
    outputs (the general store)."""
    k, n = 768, 3072
    w = tw.round_to(tw.synthetic_matrix(0, k, n, tw.STREAM_WEIGHTS), compute)
    a = tw.round_to(tw.synthetic_matrix(0, m, k, tw.STREAM_INPUT), compute)
    _, tsm, ov = tw.prune_tew(w, 0.75, 0.015, 128)
    enc = tw.encode_cto(tsm)
    p16 = tw.TwPlan(enc, ov, compute_dtype=compute)
    monkeypatch.setenv("TW_K2_TPL", "8")
    p8 = tw.TwPlan(enc, ov, compute_dtype=compute)
    x = p16.prepare(a)
    assert torch_equal(p16.run_tew(x, out_dtype=out_dtype), p8.run_tew(x, out_dtype=out_dtype))
    idx = np.arange(0, m, max(1, m // 64))
    ref, _ = orc.tew_reference(a[idx], enc, ov.col_ptr, ov.row_idx, ov.values, n)
    o32 = p16.run_tew(x, out_dtype="fp32").t().cpu().numpy()[idx]
    assert tw.relative_error(o32, ref) <= TOL["fp32"]


@pytest.mark.parametrize("k,n,m,out_dtype,env", [
    (768, 768, 700, "fp32", {}),
    (3072, 768, 500, "fp16", {}),
    (768, 3072, 300, "fp16", {"TW_RUN_COPIES": "3"}),   # G copies: K2 reads copy 0
    (768, 768, 333, "fp32", {"TW_RESIDUAL_DIRECT": "1"}),  # K2 per-entry path, remapped rows
])
def test_tew_row_runs_layout_bit_identical(k, n, m, out_dtype, env, monkeypatch):
    """TEW on a row-run plan: K1 and K2 both read A^T in the plan layout (the
    overlay rows remapped to layout positions) and give exactly the result of
    the natural-order input through the same plan; the oracle agrees."""
    for name, value in env.items():
        monkeypatch.setenv(name, value)
    rng = np.random.default_rng(k + n + m)
    w = tw.round_to(rng.normal(size=(k, n)).astype(np.float32), "fp16")
    a = tw.round_to(rng.normal(size=(m, k)).astype(np.float32), "fp16")
    _, tsm, ov = tw.prune_tew(w, 0.75, 0.015, 128)
    plan = tw.TwPlan(tw.encode_cto(tsm), ov, row_layout="runs")
    assert plan.uses_row_runs
    o_plan = plan.run_tew(plan.prepare(a), out_dtype=out_dtype)
    o_nat = plan.run_tew(tw.prepare_activations(a), out_dtype=out_dtype, x_layout="natural")
    assert torch_equal(o_plan, o_nat)
    out = tw.gemm_tew(a, tsm, ov)      # plan_for: row-run layout by default
    ref, union = orc.tew_reference(a, tw.encode_cto(tsm), ov.col_ptr, ov.row_idx, ov.values, n)
    assert np.array_equal(out.column_map.kept, union)
    assert tw.relative_error(out.condensed, ref) <= TOL["fp32"]
    assert tw.relative_error(o_plan.float().t(), ref) <= TOL[out_dtype]


def test_big_layer_full_size():
    """configs[4] at its full size (16384 x 16384 weight, TW 75 %, G = 128,
    M = 8192; 64 tiles, streamed payload, strided units): the launch is
    deterministic, 64 sampled tokens of the fp32 output match the oracle
    (fp64, reference accumulation order) and the fp16 output is the fp32 one
    rounded."""
    import torch

    k = n = 16384
    m = 8192
    w = tw.round_to(tw.synthetic_matrix(0, k, n, tw.STREAM_WEIGHTS), "fp16")
    _, tsm = tw.prune_tw(w, 0.75, 128)
    del w
    assert len(tsm.tiles) == 64 and tsm.n_condensed == 8192
    enc = tw.encode_cto(tsm)
    a = tw.round_to(tw.synthetic_matrix(0, m, k, tw.STREAM_INPUT), "fp16")
    plan = tw.TwPlan(enc)
    at = plan.prepare(torch.from_numpy(a).cuda())
    c1 = plan.run(at)
    c2 = plan.run(at)
    assert torch.equal(c1, c2)
    h = plan.run(at, out_dtype="fp16")
    assert torch.equal(h, c1.half())
    idx = np.sort(np.random.default_rng(4).choice(m, 64, replace=False))
    ref = orc.c_gemm_cto_enc(np.ascontiguousarray(a[idx]), enc)
    got = c1[:, torch.from_numpy(idx).cuda()].t().cpu().numpy()
    assert tw.relative_error(got, ref) <= TOL["fp32"]
