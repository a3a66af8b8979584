"""K1 tuning probe (diagnostics, GPU box): per-layer kernel time for a list of
environment settings (TW_TN, TW_STREAMK, TW_DEBUG_FLAGS, ...).  Each setting is
a comma-separated list of NAME=VALUE; settings are separated by ';'.

    python scripts/kprobe.py "TW_TN=256;TW_TN=192;TW_STREAMK=1;TW_DEBUG_FLAGS=1"

Times are CUDA-graph replays of `reps` back-to-back launches over 4 rotating
buffer sets (cold-ish L2).  Flags != 0 break numerics (diagnostics only).
"""

from __future__ import annotations

import argparse
import os
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2402_10876_b200 as tw  # noqa: E402

LAYERS = [(768, 768), (768, 3072), (3072, 768)]


def time_layer(plans, ats, outs, reps, nsets=4):
    g = torch.cuda.CUDAGraph()
    s_ = torch.cuda.Stream()
    s_.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s_):
        plans[0].run(ats[0], out=outs[0])
        with torch.cuda.graph(g, stream=s_):
            for i in range(reps):
                plans[i % nsets].run(ats[i % nsets], out=outs[i % nsets])
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
    ap.add_argument("settings")
    ap.add_argument("--m", type=int, default=8192)
    ap.add_argument("--reps", type=int, default=40)
    ap.add_argument("--g", type=int, default=128)
    ap.add_argument("--layers", default="0,1,2")
    ap.add_argument("--sets", type=int, default=4, help="rotating buffer sets (1 = L2-warm)")
    ap.add_argument("--pad", type=int, default=0, help="extra tokens of A^T row pitch")
    ap.add_argument("--tew", type=float, default=0.0, help="TEW delta (0 = TW)")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    layers = [LAYERS[int(i)] for i in args.layers.split(",")]
    data = []
    for k, n in layers:
        w = tw.round_to(tw.synthetic_matrix(0, k, n, 0), "fp16")
        if args.tew:
            _, tsm, ov = tw.prune_tew(w, 0.75, args.tew, args.g)
            plans = [tw.TwPlan(tw.encode_cto(tsm), overlay=ov) for _ in range(4)]
            for pl in plans:
                pl.run = pl.run_tew
        else:
            _, tsm = tw.prune_tw(w, 0.75, args.g)
            plans = [tw.TwPlan(tw.encode_cto(tsm), row_layout=os.environ.get('TW_ROW_LAYOUT', 'runs')) for _ in range(4)]
        a = tw.round_to(tw.synthetic_matrix(0, args.m, k, 1), "fp16")
        ats = [pl.prepare(torch.from_numpy(a).cuda()) for pl in plans]
        if args.pad:
            padded = []
            for at in ats:
                buf = torch.zeros((at.shape[0], at.shape[1] + args.pad), dtype=at.dtype,
                                  device=at.device)
                buf[:, :at.shape[1]] = at
                padded.append(buf[:, :at.shape[1]])
            ats = padded
        rows = plans[0].info.n_union if args.tew else tsm.n_condensed
        outs = [torch.empty((rows, args.m), dtype=torch.float16, device="cuda")
                for _ in range(4)]
        ref = plans[0].run(ats[0]).float()
        data.append((plans, ats, outs, ref))
    for setting in args.settings.split(";"):
        env = dict(kv.split("=") for kv in setting.split(",") if kv)
        saved = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        line = []
        for (k, n), (plans, ats, outs, ref) in zip(layers, data):
            err = float("nan")
            if env.get("TW_DEBUG_FLAGS", "0") == "0":
                got = plans[0].run(ats[0], out_dtype="fp32").float()
                err = (got - ref).abs().max().item() / ref.abs().max().item()
            us = time_layer(plans, ats, outs, args.reps, args.sets)
            line.append(f"{k}x{n}: {us:6.1f} us (err {err:.0e})")
        for k_, v in saved.items():
            if v is None:
                os.environ.pop(k_, None)
            else:
                os.environ[k_] = v
        print(f"{setting:40s} " + " | ".join(line), flush=True)


if __name__ == "__main__":
    main()
