"""Probe (GPU box): K4 (A -> A^T, plan row order) per BERT layer, 64x64 vs 64x128 tiles."""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2402_10876_b200 as tw  # noqa: E402
from scripts.group_probe import graph_time  # noqa: E402

m = 8192
tot = {}
for k, n in [(768, 768), (768, 3072), (3072, 768)]:
    w = tw.round_to(tw.synthetic_matrix(0, k, n, 0), "fp16")
    p = tw.TwPlan(tw.encode_cto(tw.prune_tw(w, 0.75, 128)[1]), row_layout="runs")
    a = torch.randn((m, k), device="cuda", dtype=torch.float16)
    outs = [torch.empty((p.layout_rows, m), device="cuda", dtype=torch.float16) for _ in range(4)]
    ref = p.prepare(a)
    for v in ("0", "1"):
        os.environ["TW_T64"] = v if v == "1" else ""
        if v == "0":
            os.environ.pop("TW_T64")
        assert torch.equal(p.prepare(a, out=outs[0]), ref)
        t = graph_time(lambda i: p.prepare(a, out=outs[i]))
        tot[v] = tot.get(v, 0) + t
        print(f"{k}x{n} {'64x64 ' if v == '1' else '64x128'}: {t:.1f} us, "
              f"{2 * m * k * 2 / (t * 1e-6) / 1e12:.2f} TB/s")
print("step totals us:", tot)
