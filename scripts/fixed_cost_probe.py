"""K1's fixed per-launch cost at small M (configs[0]'s 1024^2 plan, runs
layout): 32-launch CUDA graphs with parts of the kernel switched off
(TW_DEBUG_FLAGS: 1 no A loads, 2 no output stores, 4 no MMAs, 16 no payload
loads, 8 launch without programmatic dependent launch).  Diagnostic only."""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2402_10876_b200 as tw  # noqa: E402
from bench import graph_us  # noqa: E402


def main():
    k = n = 1024
    w = tw.round_to(tw.synthetic_matrix(0, k, n, tw.STREAM_WEIGHTS), "fp16")
    _, tsm = tw.prune_tw(w, 0.75, 128)
    plan = tw.TwPlan(tw.encode_cto(tsm), row_layout="runs")
    for m in (1, 128):
        a = tw.round_to(tw.synthetic_matrix(0, m, k, tw.STREAM_INPUT), "fp16")
        x = plan.prepare(torch.from_numpy(a).cuda())
        o = plan.run(x, out_dtype="fp16")
        line = [f"m={m}"]
        for flags in (0, 2, 1 | 16, 1 | 2 | 16, 1 | 2 | 4 | 16, 8, 8 | 1 | 2 | 4 | 16):
            os.environ["TW_DEBUG_FLAGS"] = str(flags)
            line.append(f"flags {flags}: {graph_us(lambda i: plan.run(x, out=o, out_dtype='fp16'), 32):.2f}")
        del os.environ["TW_DEBUG_FLAGS"]
        print(" | ".join(line), flush=True)
    # an empty kernel launched the same way (torch elementwise on 1 element)
    t = torch.zeros(1, device="cuda")
    print(f"torch 1-element add in a 32-launch graph: {graph_us(lambda i: t.add_(1), 32):.2f} us")


if __name__ == "__main__":
    main()
