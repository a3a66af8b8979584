"""K2 (TEW overlay) timing on the BERT TEW layers, for A/B runs of library
builds (TW_LIB_PATH picks the .so).  Per layer: K2 alone (TW_TEW_PARTS=2) and
K1 + K2, each as a 32-launch CUDA graph; then the grouped TEW step (all three
layers, one K1 launch + one K2 launch).  256 sampled tokens of every layer are
checked against the oracle, and a checksum of the fp16 outputs is printed so
two builds can be compared bit for bit.  Diagnostic only (GPU box).
"""
import hashlib
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2402_10876_b200 as tw  # noqa: E402
from bench import graph_us  # noqa: E402
from oracle import tilesparse_oracle as orc  # noqa: E402


def main():
    m = int(os.environ.get("M", 8192))
    layers = [(768, 768), (768, 3072), (3072, 768)]
    plans, xs, outs, line = [], [], [], []
    digest = hashlib.sha256()
    for k, n in layers:
        w = tw.round_to(tw.synthetic_matrix(0, k, n, tw.STREAM_WEIGHTS), "fp16")
        a = tw.round_to(tw.synthetic_matrix(0, m, k, tw.STREAM_INPUT), "fp16")
        _, tsm, ov = tw.prune_tew(w, 0.75, 0.015, 128)
        enc = tw.encode_cto(tsm)
        layout = "runs" if os.environ.get("RUNS") == "1" else "natural"
        plan = tw.TwPlan(enc, ov, row_layout=layout)
        x = plan.prepare(a)
        o = plan.run_tew(x, out_dtype="fp16")
        torch.cuda.synchronize()
        digest.update(o.cpu().numpy().tobytes())
        both = graph_us(lambda i: plan.run_tew(x, out=o, out_dtype="fp16"), 32)
        os.environ["TW_TEW_PARTS"] = "2"
        alone = graph_us(lambda i: plan.run_tew(x, out=o, out_dtype="fp16"), 32)
        os.environ["TW_TEW_PARTS"] = "1"
        k1 = graph_us(lambda i: plan.run_tew(x, out=o, out_dtype="fp16"), 32)
        del os.environ["TW_TEW_PARTS"]
        tw_plan = tw.TwPlan(enc, row_layout=layout)
        xt = tw_plan.prepare(a)
        ot = tw_plan.run(xt, out_dtype="fp16")
        k1_tw = graph_us(lambda i: tw_plan.run(xt, out=ot, out_dtype="fp16"), 32)
        o32 = plan.run_tew(x, out_dtype="fp32")
        idx = np.arange(0, m, max(1, m // 256))
        ref, _ = orc.tew_reference(a[idx], enc, ov.col_ptr, ov.row_idx, ov.values, n)
        err = tw.relative_error(o32.t()[torch.as_tensor(idx, device=o32.device)].cpu().numpy(), ref)
        line.append(f"{k}x{n} runs={int(plan.uses_row_runs)}/{int(tw_plan.uses_row_runs)}: "
                    f"K1 {k1:.2f} (TW plan {k1_tw:.2f}) us, K2 {alone:.2f} us, "
                    f"K1+K2 {both:.2f} us, rel err {err:.2e}")
        plans.append(plan)
        xs.append(x)
        outs.append(o)
    group = tw.TwPlanGroup(plans, m)
    group.run_tew(xs, outs, out_dtype="fp16")
    step = graph_us(lambda i: group.run_tew(xs, outs, out_dtype="fp16"), 16)
    print(" | ".join(line) + f" | grouped TEW step {step:.2f} us | sha {digest.hexdigest()[:16]}",
          flush=True)


if __name__ == "__main__":
    main()
