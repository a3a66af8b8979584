"""One sparse and one dense K1 launch of the BERT 768x768 TVW layer (natural
row order, owner mode) for an ncu comparison (-k regex:tw_gemm)."""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2402_10876_b200 as tw  # noqa: E402

k, n = (int(v) for v in os.environ.get("LAYER", "768x768").split("x"))
m = 8192
w = tw.round_to(tw.synthetic_matrix(0, k, n, tw.STREAM_WEIGHTS), "fp16")
a = tw.round_to(tw.synthetic_matrix(0, m, k, tw.STREAM_INPUT), "fp16")
_, tsm, _ = tw.prune_tvw(w, 0.75, 128)
plan = tw.TwPlan(tw.encode_cto(tsm), row_layout="natural")
x = plan.prepare(a)
os.environ["TW_OWNER"] = "1"
for ns in ("0", "1"):
    os.environ["TW_NO_SPARSE"] = ns
    plan.run(x, out_dtype="fp16")
    torch.cuda.synchronize()
