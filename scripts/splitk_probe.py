"""Split-K for small M (tw_capi.cu, kSplitKMaxTokens): K1 per launch with
TW_SPLITK=0 (one CTA streams every stage of its sub-tile) against the
split-K path (TW_SPLITK=1: the stages over several CTAs + splitk_reduce), on
the BERT shapes and configs[0]'s 1024^2, fp32 out, against the oracle.
Diagnostic only (GPU box): python scripts/splitk_probe.py
"""
import os, sys
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2402_10876_b200 as tw
from oracle import tilesparse_oracle as orc
from bench import graph_us
for (k, n) in [(1024, 1024), (768, 3072), (3072, 768)]:
    w = tw.round_to(tw.synthetic_matrix(0, k, n, tw.STREAM_WEIGHTS), "fp16")
    _, tsm = tw.prune_tw(w, 0.75, 128)
    enc = tw.encode_cto(tsm)
    for layout in ("natural", "runs"):
        plan = tw.TwPlan(enc, row_layout=layout)
        for m in (1, 17, 128, 200, 256, 300):
            a = tw.round_to(tw.synthetic_matrix(0, m, k, tw.STREAM_INPUT), "fp16")
            x = plan.prepare(torch.from_numpy(a).cuda())
            os.environ["TW_SPLITK"] = "0"
            o0 = plan.run(x, out_dtype="fp32"); torch.cuda.synchronize()
            t0 = graph_us(lambda i: plan.run(x, out=o0, out_dtype="fp32"), 32)
            os.environ["TW_SPLITK"] = "1"
            o1 = plan.run(x, out_dtype="fp32"); torch.cuda.synchronize()
            t1 = graph_us(lambda i: plan.run(x, out=o1, out_dtype="fp32"), 32)
            h1 = plan.run(x, out_dtype="fp16"); torch.cuda.synchronize()
            ref = orc.c_gemm_cto_enc(a, enc)
            e1 = tw.relative_error(o1.t().cpu().numpy(), ref)
            e0 = tw.relative_error(o0.t().cpu().numpy(), ref)
            eh = tw.relative_error(h1.float().t().cpu().numpy(), ref)
            print(f"{k}x{n} {layout:7s} m={m:4d} no-split {t0:6.2f} us err {e0:.1e} | split {t1:6.2f} us err {e1:.1e} fp16 {eh:.1e}", flush=True)
