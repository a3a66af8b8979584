"""configs[3]: VGG-16 conv layers as im2col GEMMs, batch 64, TW sparsity sweep.

    python scripts/vgg_sweep.py [--s 0.5,0.6,0.7,0.8,0.9] [--g 64,128,256]
                                [--layers all|conv4_2,...] [--out FILE]

Per conv layer (M = 64*H*W tokens, K = 9*C_in, N = C_out) and per (s, G):
prune the synthetic weight on the host (prune_tw, bit-exact with the
reference), build the device plan, and time K1 (CUDA events over a graph of
back-to-back launches) against dense cuBLAS at the same shape and layout
(C^T = W^T . A^T).  Activations are random fp16 generated on the device (the
im2col matrices of conv1_x are 3.2M x 576: too large to draw on the host);
correctness at these shapes is covered by tests/test_gpu_parity.py.
Prints one JSON object with a row per (layer, s, G).
"""

from __future__ import annotations

import argparse
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2402_10876_b200 as tw  # noqa: E402

# name: (H=W of the output map, C_in, C_out); batch 64, 3x3 kernels, pad 1
VGG16 = {
    "conv1_1": (224, 3, 64), "conv1_2": (224, 64, 64),
    "conv2_1": (112, 64, 128), "conv2_2": (112, 128, 128),
    "conv3_1": (56, 128, 256), "conv3_2": (56, 256, 256), "conv3_3": (56, 256, 256),
    "conv4_1": (28, 256, 512), "conv4_2": (28, 512, 512), "conv4_3": (28, 512, 512),
    "conv5_1": (14, 512, 512), "conv5_2": (14, 512, 512), "conv5_3": (14, 512, 512),
}
BATCH = 64


def shape(name: str):
    hw, cin, cout = VGG16[name]
    return BATCH * hw * hw, 9 * cin, cout  # M, K, N


def time_graph(fn, reps: int) -> float:
    """Median per-call microseconds of `reps` back-to-back calls in a graph."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        fn()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / reps)
    return statistics.median(ts)


def run(layers, sparsities, gs, reps_for=lambda m: 20 if m < 1_000_000 else 5):
    rows = []
    for name in layers:
        m, k, n = shape(name)
        at = (torch.randn((k, m), device="cuda", dtype=torch.float16))
        w = tw.round_to(tw.synthetic_matrix(0, k, n, tw.STREAM_WEIGHTS), "fp16")
        wt = torch.from_numpy(w.T.copy()).to("cuda", torch.float16)
        dense = torch.empty((n, m), device="cuda", dtype=torch.float16)
        reps = reps_for(m)
        us_dense = time_graph(lambda: torch.matmul(wt, at, out=dense), reps)
        del dense
        for g in gs:
            for s in sparsities:
                _, tsm = tw.prune_tw(w, s, g)
                plan = tw.TwPlan(tw.encode_cto(tsm), row_layout="runs")
                x = plan.prepare(at=at) if plan.uses_row_runs else at   # plan row order
                out = torch.empty((tsm.n_condensed, m), device="cuda", dtype=torch.float16)
                us = time_graph(lambda: plan.run(x, out=out), reps)
                # the row-run path must equal the natural-order gather bit for bit
                same = None
                if plan.uses_row_runs:
                    nat = plan.run(at, out_dtype="fp16", x_layout="natural")
                    same = bool(torch.equal(out, nat))
                    del nat
                flops = tw.sparse_flops(tsm, m)
                rows.append({"layer": name, "M": m, "K": k, "N": n, "s": s, "g": g,
                             "n_tiles": len(tsm.tiles), "n_condensed": int(tsm.n_condensed),
                             "row_runs": bool(plan.uses_row_runs), "runs_bit_identical": same,
                             "kept_rows_min": min(t.kept_rows.n_kept for t in tsm.tiles),
                             "us": us, "us_cublas": us_dense, "speedup": us_dense / us,
                             "tflops_effective": flops / (us * 1e-6) / 1e12,
                             "tflops_cublas_dense": 2 * m * k * n / (us_dense * 1e-6) / 1e12})
                del plan, out, x
        del at, wt
        torch.cuda.empty_cache()
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--s", default="0.5,0.6,0.7,0.8,0.9")
    ap.add_argument("--g", default="64,128,256")
    ap.add_argument("--layers", default="all")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    layers = list(VGG16) if args.layers == "all" else args.layers.split(",")
    rows = run(layers, [float(x) for x in args.s.split(",")], [int(x) for x in args.g.split(",")])
    doc = {"config": "VGG-16 im2col GEMMs, batch 64, fp16, TW sweep (configs[3])",
           "device": torch.cuda.get_device_name(), "rows": rows}
    text = json.dumps(doc, indent=1)
    if args.out:
        Path(args.out).write_text(text)
    bad = [r for r in rows if r["runs_bit_identical"] is False]
    if bad:
        print(f"ERROR: {len(bad)} points differ between the run path and the gather")
    for r in rows:
        print(f"{r['layer']:8s} s={r['s']:.1f} g={r['g']:3d} tiles={r['n_tiles']:2d} "
              f"K'min={r['kept_rows_min']:4d} {r['us']:9.1f} us  cuBLAS {r['us_cublas']:9.1f} us  "
              f"x{r['speedup']:.2f}  {r['tflops_effective']:.0f} TF/s")


if __name__ == "__main__":
    main()
