"""One TEW launch (K1 + K2) on a BERT TEW layer, for an ncu capture of K2
(-k regex:tw_residual).  LAYER=768x3072 by default."""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2402_10876_b200 as tw  # noqa: E402

k, n = (int(v) for v in os.environ.get("LAYER", "768x3072").split("x"))
m = 8192
w = tw.round_to(tw.synthetic_matrix(0, k, n, tw.STREAM_WEIGHTS), "fp16")
a = tw.round_to(tw.synthetic_matrix(0, m, k, tw.STREAM_INPUT), "fp16")
_, tsm, ov = tw.prune_tew(w, 0.75, 0.015, 128)
plan = tw.TwPlan(tw.encode_cto(tsm), ov)
x = plan.prepare(a)
plan.run_tew(x, out_dtype="fp16")
torch.cuda.synchronize()
