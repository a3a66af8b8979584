"""Seeded random problems through every K1 mode (GPU).

Each case draws a shape, sparsity, tile width, token count and one set of
mode switches (owner / strided, resident / streamed payload, row-run layout
with one or grouped copies, the cp.async gather by layout position), then
checks that

* two launches give the same bits (no races),
* the row-run layout gives exactly the bits of the natural-order gather
  through the same plan,
* the result matches the CPU oracle within the fp32 / fp16 / bf16 tolerance.

This is the test that would have caught the resident run-path epilogue bug
fixed in round 1.
"""

from __future__ import annotations

import numpy as np
import pytest

import paper_2402_10876_b200 as tw
from oracle import tilesparse_oracle as orc

pytestmark = pytest.mark.gpu

TOL = {"fp32": 1e-5, "fp16": 1e-3, "bf16": 8e-3}
MODES = [{}, {"TW_STRIDED": "1"}, {"TW_OWNER": "1"}, {"TW_NO_RESIDENT": "1"},
         {"TW_RUN_COPIES": "3"}, {"TW_RUN_MAX_UNITS": "0"}, {"TW_RUN_COPIES": "2", "TW_STRIDED": "1"}]


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    k = int(rng.choice([64, 200, 512, 768, 1000, 1536, 3072]))
    n = int(rng.choice([96, 256, 640, 768, 1536, 3072]))
    m = int(rng.choice([1, 17, 300, 1000, 4097, 8192, 16384]))
    s = float(rng.choice([0.5, 0.6, 0.75, 0.8, 0.9]))
    g = int(rng.choice([32, 64, 128, 256]))
    dt = str(rng.choice(["fp16", "bf16"]))
    out = str(rng.choice(["fp32", "fp16" if dt == "fp16" else "bf16"]))
    mode = MODES[seed % len(MODES)]
    return k, n, m, s, g, dt, out, mode, rng


@pytest.mark.parametrize("seed", range(49))
def test_random_problem(seed, monkeypatch):
    k, n, m, s, g, dt, out_dt, mode, rng = _case(seed)
    for key, v in mode.items():
        monkeypatch.setenv(key, v)
    w = tw.round_to(rng.normal(size=(k, n)).astype(np.float32), dt)
    a = tw.round_to(rng.normal(size=(m, k)).astype(np.float32), dt)
    _, tsm = tw.prune_tw(w, s, g)
    enc = tw.encode_cto(tsm)
    plan = tw.TwPlan(enc, compute_dtype=dt, row_layout="runs")
    x = plan.prepare(a)
    o1 = plan.run(x, out_dtype=out_dt)
    o2 = plan.run(x, out_dtype=out_dt)
    assert bool((o1 == o2).all()), f"non-deterministic: {k}x{n} m={m} g={g} {mode}"
    if plan.uses_row_runs:
        nat = plan.run(tw.prepare_activations(a, dt), out_dtype=out_dt, x_layout="natural")
        assert bool((o1 == nat).all()), f"run path != gather: {k}x{n} m={m} g={g} {mode}"
    ref = orc.c_gemm_cto_enc(a, enc, threads=8)
    err = tw.relative_error(o1.float().t(), ref)
    assert err <= TOL[out_dt if out_dt == "fp32" else dt], (k, n, m, s, g, dt, out_dt, mode, err)
