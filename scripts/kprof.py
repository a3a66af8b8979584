"""Kernel timing probe (GPU box): per-layer K1 time for each gather mode and
diagnostic flag set.  Results are for tuning only (flags break numerics).

    python scripts/kprof.py [--modes 0,1] [--flags 0,1,2,4] [--m 8192]
"""

from __future__ import annotations

import argparse
import os
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2402_10876_b200 as tw  # noqa: E402

LAYERS = [(768, 768), (768, 3072), (3072, 768)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--modes", default="0,1")
    ap.add_argument("--flags", default="0,1,2,4")
    ap.add_argument("--m", type=int, default=8192)
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--g", type=int, default=128)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    plans, ats, outs = [], [], []
    for k, n in LAYERS:
        w = tw.round_to(tw.synthetic_matrix(0, k, n, 0), "fp16")
        _, tsm = tw.prune_tw(w, 0.75, args.g)
        plans.append([tw.TwPlan(tw.encode_cto(tsm), row_layout=os.environ.get('TW_ROW_LAYOUT', 'runs')) for _ in range(4)])
        a = tw.round_to(tw.synthetic_matrix(0, args.m, k, 1), "fp16")
        ats.append([pl.prepare(torch.from_numpy(a).cuda()) for pl in plans[-1]])
        outs.append([torch.empty((tsm.n_condensed, args.m), dtype=torch.float16, device="cuda")
                     for _ in range(4)])
    ref = [plans[i][0].run(ats[i][0]).float() for i in range(3)]
    for mode in [int(x) for x in args.modes.split(",")]:
        for flags in [int(x) for x in args.flags.split(",")]:
            os.environ["TW_GATHER"] = str(mode)
            os.environ["TW_DEBUG_FLAGS"] = str(flags)
            line = []
            for li in range(3):
                if flags == 0:
                    got = plans[li][0].run(ats[li][0]).float()
                    err = (got - ref[li]).abs().max().item() / ref[li].abs().max().item()
                else:
                    err = float("nan")
                # CUDA graph of `reps` back-to-back launches (rotating buffers) so the
                # device never waits on the host; per-launch time = graph time / reps
                g = torch.cuda.CUDAGraph()
                s_ = torch.cuda.Stream()
                s_.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(s_):
                    plans[li][0].run(ats[li][0], out=outs[li][0])
                    with torch.cuda.graph(g, stream=s_):
                        for i in range(args.reps):
                            plans[li][i % 4].run(ats[li][i % 4], out=outs[li][i % 4])
                torch.cuda.current_stream().wait_stream(s_)
                g.replay()
                torch.cuda.synchronize()
                times = []
                for _ in range(5):
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record()
                    g.replay()
                    e1.record()
                    torch.cuda.synchronize()
                    times.append(e0.elapsed_time(e1) * 1e3 / args.reps)
                us = statistics.median(times)
                if os.environ.get("KPROF_VERBOSE"):
                    print(f"  mode={mode} flags={flags} layer {li}: {us:.1f} us", flush=True)
                line.append(f"{LAYERS[li][0]}x{LAYERS[li][1]}: {us:7.1f} us (err {err:.1e})")
            print(f"mode={mode} flags={flags}: " + " | ".join(line), flush=True)
    os.environ.pop("TW_DEBUG_FLAGS", None)
    os.environ.pop("TW_GATHER", None)


if __name__ == "__main__":
    main()
