"""Probe (GPU box): K1 on the TW plan vs K1 on a 'row-densified' plan of the
same layer (every tile keeps all K rows, pruned payload rows zero) vs dense
cuBLAS on the column-condensed weight (K x N') and on the full weight.

    python scripts/densify_probe.py [--m 8192]
"""

from __future__ import annotations

import argparse
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2402_10876_b200 as tw  # noqa: E402
from paper_2402_10876_b200.core import IndexMask  # noqa: E402
from paper_2402_10876_b200.patterns import Tile, TileSparseMatrix  # noqa: E402

LAYERS = [(768, 768), (768, 3072), (3072, 768)]


def densify(tsm: TileSparseMatrix) -> TileSparseMatrix:
    k = tsm.original_dims[0]
    tiles = []
    for t in tsm.tiles:
        p = np.zeros((k, t.width), np.float32)
        p[t.kept_rows.kept] = t.payload
        tiles.append(Tile(IndexMask(k, np.arange(k)), p))
    return TileSparseMatrix(tsm.config, tsm.column_mask, tuple(tiles), tsm.original_dims)


def time_graph(fn, reps=32):
    g = torch.cuda.CUDAGraph()
    s_ = torch.cuda.Stream()
    s_.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s_):
        fn(0)
        with torch.cuda.graph(g, stream=s_):
            for i in range(reps):
                fn(i)
    torch.cuda.current_stream().wait_stream(s_)
    g.replay()
    torch.cuda.synchronize()
    times = []
    for _ in range(7):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) * 1e3 / reps)
    return statistics.median(times)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=8192)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    for k, n in LAYERS:
        w = tw.round_to(tw.synthetic_matrix(0, k, n, 0), "fp16")
        _, tsm = tw.prune_tw(w, 0.75, 128)
        a = tw.round_to(tw.synthetic_matrix(0, args.m, k, 1), "fp16")
        a_d = torch.from_numpy(a).cuda()
        res = {}
        outs = {}
        for name, t in (("tw", tsm), ("dense_k", densify(tsm))):
            for layout in ("runs", "natural"):
                plans = [tw.TwPlan(tw.encode_cto(t), row_layout=layout) for _ in range(4)]
                ats = [pl.prepare(a_d) for pl in plans]
                cts = [torch.empty((t.n_condensed, args.m), dtype=torch.float16, device="cuda")
                       for _ in range(4)]
                us = time_graph(lambda i: plans[i % 4].run(ats[i % 4], out=cts[i % 4]))
                outs[(name, layout)] = plans[0].run(ats[0]).float()
                res[f"{name}/{layout}"] = us
        ref = outs[("tw", "runs")]
        errs = {f"{a}/{b}": ((o - ref).abs().max() / ref.abs().max()).item()
                for (a, b), o in outs.items()}
        wc = torch.from_numpy(w[:, tsm.column_mask.kept]).cuda().half()
        wf = torch.from_numpy(w).cuda().half()
        ah = [a_d.half().clone() for _ in range(4)]
        res["cublas_cond"] = time_graph(lambda i: torch.matmul(ah[i % 4], wc))
        res["cublas_full"] = time_graph(lambda i: torch.matmul(ah[i % 4], wf))
        print(f"{k}x{n} tiles={len(tsm.tiles)} N'={tsm.n_condensed}: "
              + " ".join(f"{kk}={v:.1f}us" for kk, v in res.items())
              + " errs " + " ".join(f"{kk}={v:.1e}" for kk, v in errs.items()), flush=True)


if __name__ == "__main__":
    main()
