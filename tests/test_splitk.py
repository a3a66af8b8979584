"""Split-K for small M (tw_capi.cu, kSplitKMaxTokens / kSplitKMinSteps): the
k-steps of every sub-tile spread over several CTAs, fp32 partial products in
the plan's workspace, summed in split order by splitk_reduce.  Checked
against the oracle (fp64) and against the single-CTA-per-sub-tile path
(TW_SPLITK=0), for TW and TEW, both input layouts and the 16-bit and fp32
outputs.  Tolerances as in test_gpu_parity.py.
"""

from __future__ import annotations

import numpy as np
import pytest

import paper_2402_10876_b200 as tw
from oracle import tilesparse_oracle as orc

pytestmark = pytest.mark.gpu

TOL = {"fp32": 1e-5, "fp16": 1e-3, "bf16": 8e-3}


def _layer(k, n, compute, tew=False):
    w = tw.round_to(tw.synthetic_matrix(0, k, n, tw.STREAM_WEIGHTS), compute)
    if tew:
        _, tsm, ov = tw.prune_tew(w, 0.75, 0.015, 128)
        return tsm, ov
    _, tsm = tw.prune_tw(w, 0.75, 128)
    return tsm, None


@pytest.mark.parametrize("m", [1, 37, 128, 129])
@pytest.mark.parametrize("layout", ["natural", "runs"])
@pytest.mark.parametrize("compute,out_dtype", [("fp16", "fp32"), ("fp16", "fp16"),
                                               ("bf16", "bf16")])
def test_splitk_tw_matches_oracle(m, layout, compute, out_dtype, monkeypatch):
    """3072 x 768 (43 k-steps per sub-tile): split-K for M <= 128, the
    regular path at 129; both agree with the oracle and with each other."""
    import torch

    k, n = 3072, 768
    tsm, _ = _layer(k, n, compute)
    enc = tw.encode_cto(tsm)
    plan = tw.TwPlan(enc, compute_dtype=compute, row_layout=layout)
    a = tw.round_to(tw.synthetic_matrix(0, m, k, tw.STREAM_INPUT), compute)
    x = plan.prepare(a)
    out = plan.run(x, out_dtype=out_dtype)
    ref = orc.c_gemm_cto_enc(a, enc)
    assert tw.relative_error(out.float().t().cpu().numpy(), ref) <= TOL[out_dtype]
    monkeypatch.setenv("TW_SPLITK", "0")
    single = plan.run(x, out_dtype="fp32")
    torch.cuda.synchronize()
    assert tw.relative_error(out.float().t().cpu().numpy(),
                             single.t().cpu().numpy()) <= TOL[out_dtype]


@pytest.mark.parametrize("m", [5, 96])
def test_splitk_tew_matches_oracle(m):
    """TEW at small M: K1 split-K into the workspace (condensed rows) or
    straight onto the union rows (rowmap in splitk_reduce), then K2."""
    import torch

    from paper_2402_10876_b200 import _native

    k, n = 3072, 768
    tsm, ov = _layer(k, n, "fp16", tew=True)
    enc = tw.encode_cto(tsm)
    plan = tw.TwPlan(enc, ov)
    a = tw.round_to(tw.synthetic_matrix(0, m, k, tw.STREAM_INPUT), "fp16")
    x = plan.prepare(a)
    ref, union = orc.tew_reference(a, enc, ov.col_ptr, ov.row_idx, ov.values, n)
    o_ws = plan.run_tew(x, out_dtype="fp32")
    assert tw.relative_error(o_ws.t().cpu().numpy(), ref) <= TOL["fp32"]
    o_sc = torch.empty_like(o_ws)
    lib = _native.load_library()
    _native.check(lib.tw_gemm_tew(plan._handle, x.data_ptr(), x.shape[1], x.stride(0),
                                  o_sc.data_ptr(), o_sc.stride(0), _native.TW_F32,
                                  _native.stream_handle()))
    torch.cuda.synchronize()
    assert tw.relative_error(o_sc.t().cpu().numpy(), ref) <= TOL["fp32"]


def test_splitk_deterministic_and_group_path_unsplit():
    """Repeated split-K launches are bit-identical (fixed split order), and a
    TwPlanGroup launch (one kernel for all plans, never split) agrees within
    the fp32 tolerance."""
    import torch

    k, n, m = 3072, 768, 64
    tsm, _ = _layer(k, n, "fp16")
    plan = tw.TwPlan(tw.encode_cto(tsm), row_layout="runs")
    a = tw.round_to(tw.synthetic_matrix(0, m, k, tw.STREAM_INPUT), "fp16")
    x = plan.prepare(a)
    o1 = plan.run(x, out_dtype="fp32")
    o2 = plan.run(x, out_dtype="fp32")
    torch.cuda.synchronize()
    assert torch.equal(o1, o2)
    g = tw.TwPlanGroup([plan], m)
    (og,) = g.run([x], out_dtype="fp32", fused=True)
    torch.cuda.synchronize()
    assert tw.relative_error(og.t().cpu().numpy(), o1.t().cpu().numpy()) <= TOL["fp32"]
