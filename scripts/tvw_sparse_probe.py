"""TVW on tcgen05.mma.sp vs the dense tensor-core path (TW_NO_SPARSE=1) on
the BERT TVW layers: per-launch time in a 32-launch CUDA graph and the error
against the oracle on sampled tokens.  Diagnostic (GPU box)."""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2402_10876_b200 as tw  # noqa: E402
from oracle import tilesparse_oracle as orc  # noqa: E402
from bench import graph_us  # noqa: E402


def main():
    m = 8192
    for k, n in [(768, 768), (768, 3072), (3072, 768)]:
        w = tw.round_to(tw.synthetic_matrix(0, k, n, tw.STREAM_WEIGHTS), "fp16")
        a = tw.round_to(tw.synthetic_matrix(0, m, k, tw.STREAM_INPUT), "fp16")
        _, tsm, _ = tw.prune_tvw(w, 0.75, 128)
        enc = tw.encode_cto(tsm)
        res = []
        for layout in ("natural", "runs"):
            os.environ.pop("TW_NO_SPARSE", None)
            if layout == "runs":
                os.environ["TW_NO_SPARSE"] = "1"  # plan-time: keep the row-run layout
            plan = tw.TwPlan(enc, row_layout=layout)
            x = plan.prepare(a)
            for ns in ("0", "1", "res"):
                os.environ["TW_NO_SPARSE"] = "0" if ns == "res" else ns
                os.environ["TW_SPARSE_RESIDENT"] = "1" if ns == "res" else "0"
                if layout == "runs" and ns != "1":
                    continue
                out = plan.run(x, out_dtype="fp16")
                us = graph_us(lambda i: plan.run(x, out=out, out_dtype="fp16"), 32)
                o32 = plan.run(x, out_dtype="fp32")
                idx = np.arange(0, m, 61)
                ref = orc.c_gemm_cto_enc(a[idx], enc, threads=8)
                err = tw.relative_error(o32.t()[torch.as_tensor(idx, device=o32.device)].cpu().numpy(), ref)
                res.append(f"{layout}/sparse_plan={plan.info.sparse_payload}/no_sparse={ns}: "
                           f"{us:.2f}us err={err:.1e}")
        os.environ.pop("TW_NO_SPARSE", None)
        print(f"{k}x{n} K'max={max(t.kept_rows.n_kept for t in tsm.tiles)} | " + " | ".join(res),
              flush=True)


if __name__ == "__main__":
    main()
