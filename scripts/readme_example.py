"""The README's usage example, run as written (GPU box)."""
import numpy as np
import torch

import paper_2402_10876_b200 as tw

w = tw.round_to(np.random.default_rng(0).normal(size=(768, 3072)).astype(np.float32), "fp16")
a = tw.round_to(np.random.default_rng(1).normal(size=(8192, 768)).astype(np.float32), "fp16")
masks, tsm = tw.prune_tw(w, 0.75, 128)
enc = tw.encode_cto(tsm)
out = tw.gemm_cto(a, enc)
y = out.expand()
p = tw.TwPlan(enc, row_layout="runs")
x = p.prepare(torch.from_numpy(a).cuda())
ct = p.run(x, out_dtype="fp16")
group = tw.TwPlanGroup([p], m=8192)
(g_out,) = group.run([x], out_dtype="fp16")
torch.cuda.synchronize()
print("README example ok:", tuple(y.shape), tuple(ct.shape), torch.equal(ct, g_out))
