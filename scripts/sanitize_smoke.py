"""Small TW + TEW + transpose run for compute-sanitizer (GPU box):

    compute-sanitizer --tool memcheck|racecheck|synccheck python scripts/sanitize_smoke.py

Covers the resident (K' <= 448) and streamed K1 kernels in owner and strided
modes, ragged M / widths, 16-bit and fp32 outputs, K2 and both K4 paths, and
the row-run layout: streamed and resident payload with 3-4 units per CTA (the
last unit's epilogue joined by the idle gather warps), grouped copies, and the
cp.async gather by layout position.
"""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2402_10876_b200 as tw  # noqa: E402


def main():
    only = sys.argv[1] if len(sys.argv) > 1 else "all"   # all | small | runs | gather | k2
    rng = np.random.default_rng(0)
    if only == "k2":
        k2_and_splitk(rng)
        return
    for (k, n, m, s, g) in ([] if only in ("runs", "gather") else [(256, 384, 300, 0.75, 128), (1024, 512, 200, 0.5, 128),
                            (96, 80, 37, 0.3, 16)]):
        w = tw.round_to(rng.standard_normal((k, n)).astype(np.float32), "fp16")
        a = tw.round_to(rng.standard_normal((m, k)).astype(np.float32), "fp16")
        _, tsm = tw.prune_tw(w, s, g)
        for od in ("fp32", "fp16"):
            tw.gemm_tile_sparse(a, tsm, out_dtype=od)
        os.environ["TW_STRIDED"] = "1"
        tw.TwPlan(tw.encode_cto(tsm)).run(tw.prepare_activations(a))
        del os.environ["TW_STRIDED"]
        _, ttsm, ov = tw.prune_tew(w, s, 0.02, g)
        tw.gemm_tew(a, ttsm, ov, out_dtype="fp16")
        tw.prepare_activations(torch.from_numpy(a).cuda().half())
    # row-run layout, several units per CTA
    cases = [(768, 768, 16384, {}), (768, 3072, 8192, {"TW_RUN_COPIES": "3"}),
             (768, 768, 16384, {"TW_RUN_MAX_UNITS": "0"})]
    if only == "runs":
        cases = cases[:2]
    elif only == "gather":
        cases = cases[2:]
    elif only == "small":
        cases = []
    for (k, n, m, env) in cases:
        os.environ.update(env)
        w = tw.round_to(rng.standard_normal((k, n)).astype(np.float32), "fp16")
        a = tw.round_to(rng.standard_normal((m, k)).astype(np.float32), "fp16")
        _, tsm = tw.prune_tw(w, 0.75, 128)
        plan = tw.TwPlan(tw.encode_cto(tsm), row_layout="runs")
        plan.run(plan.prepare(a), out_dtype="fp16")
        for key in env:
            del os.environ[key]
    torch.cuda.synchronize()
    print("sanitize smoke done")


def k2_and_splitk(rng):
    """K2 with 16 tokens per lane (T = 64) and the 16-byte group loads (T =
    32), whole and ragged blocks, 16-bit and fp32 outputs, the grouped K2
    launch; split-K K1 + splitk_reduce for TW (both layouts) and TEW."""
    plans, xs = [], []
    for (k, n, m, dt) in [(768, 512, 200, "fp16"), (3072, 384, 96, "bf16"), (768, 640, 128, "fp16")]:
        w = tw.round_to(rng.standard_normal((k, n)).astype(np.float32), dt)
        a = tw.round_to(rng.standard_normal((m, k)).astype(np.float32), dt)
        _, tsm, ov = tw.prune_tew(w, 0.75, 0.015, 128)
        plan = tw.TwPlan(tw.encode_cto(tsm), ov, compute_dtype=dt, row_layout="runs")
        x = plan.prepare(a)
        for od in ("fp32", dt):
            plan.run_tew(x, out_dtype=od)
        if m == 128:
            plans.append(plan)
            xs.append(x)
    w = tw.round_to(rng.standard_normal((3072, 768)).astype(np.float32), "fp16")
    _, tsm, ov = tw.prune_tew(w, 0.75, 0.015, 128)
    p3 = tw.TwPlan(tw.encode_cto(tsm), ov, row_layout="runs")
    x3 = p3.prepare(tw.round_to(rng.standard_normal((128, 3072)).astype(np.float32), "fp16"))
    tw.TwPlanGroup(plans + [p3], 128).run_tew(xs + [x3], out_dtype="fp16")
    # split-K: 3072-row tiles (>= 16 stages), M <= 128
    _, tsm = tw.prune_tw(w, 0.75, 128)
    for layout in ("natural", "runs"):
        plan = tw.TwPlan(tw.encode_cto(tsm), row_layout=layout)
        for m in (1, 77):
            a = tw.round_to(rng.standard_normal((m, 3072)).astype(np.float32), "fp16")
            x = plan.prepare(a)
            plan.run(x, out_dtype="fp16")
            plan.run(x, out_dtype="fp32")
    p3.run_tew(x3, out_dtype="fp16")
    torch.cuda.synchronize()
    print("sanitize k2 / split-K done")


if __name__ == "__main__":
    main()
