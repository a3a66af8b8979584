"""K2m (tensor-core TEW residual) vs K2 (CUDA-core) on the BERT TEW layers.

Per layer: K2 alone (TW_TEW_PARTS=2) and K1 + K2 timed in a 32-launch CUDA
graph for both kernels (TW_K2_LEGACY selects per launch), the two results
compared with each other and sampled tokens against the oracle.
Diagnostic only (python scripts/k2m_probe.py on a GPU box).  K2m was
reverted; apply profiles/r2_k2m_experiment.patch first (it restores
TW_K2_LEGACY and the K2m kernel).
"""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2402_10876_b200 as tw  # noqa: E402
from oracle import tilesparse_oracle as orc  # noqa: E402


def timed(fn, reps=32):
    from bench import graph_us

    return graph_us(lambda i: fn(), reps)


def main():
    m = int(os.environ.get("M", 8192))
    layers = [(768, 768), (768, 3072), (3072, 768)]
    for k, n in layers:
        w = tw.round_to(tw.synthetic_matrix(0, k, n, tw.STREAM_WEIGHTS), "fp16")
        a = tw.round_to(tw.synthetic_matrix(0, m, k, tw.STREAM_INPUT), "fp16")
        _, tsm, ov = tw.prune_tew(w, 0.75, 0.015, 128)
        plan = tw.TwPlan(tw.encode_cto(tsm), ov)
        x = plan.prepare(a)
        outs, times = {}, {}
        for name, legacy in (("K2", "1"), ("K2m", "0")):
            os.environ["TW_K2_LEGACY"] = legacy
            o = plan.run_tew(x, out_dtype="fp16")
            torch.cuda.synchronize()
            outs[name] = o.float().clone()
            times[name + " k1+k2"] = timed(lambda: plan.run_tew(x, out=o, out_dtype="fp16"))
            os.environ["TW_TEW_PARTS"] = "2"
            times[name + " alone"] = timed(lambda: plan.run_tew(x, out=o, out_dtype="fp16"))
            del os.environ["TW_TEW_PARTS"]
        os.environ["TW_K2_LEGACY"] = "0"
        o32 = plan.run_tew(x, out_dtype="fp32")
        idx = np.arange(0, m, max(1, m // 256))
        ref, _ = orc.tew_reference(a[idx], tw.encode_cto(tsm), ov.col_ptr, ov.row_idx, ov.values, n)
        err = tw.relative_error(o32.t()[torch.as_tensor(idx, device=o32.device)].cpu().numpy(), ref)
        diff = (outs["K2"] - outs["K2m"]).abs().max().item()
        nnz = ov.nnz
        print(f"{k}x{n} nnz={nnz} " + " ".join(f"{kk}={v:.2f}us" for kk, v in times.items())
              + f" | fp16 max|K2-K2m|={diff:.3e} fp32 rel err vs oracle={err:.2e}"
              + f" | K2m {2 * m * nnz / times['K2m alone'] / 1e6:.1f} TFLOP/s", flush=True)




def ablate():
    """K2m alone on each layer with parts switched off (TW_DEBUG_FLAGS)."""
    m = 8192
    for k, n in [(768, 768), (768, 3072)]:
        w = tw.round_to(tw.synthetic_matrix(0, k, n, tw.STREAM_WEIGHTS), "fp16")
        a = tw.round_to(tw.synthetic_matrix(0, m, k, tw.STREAM_INPUT), "fp16")
        _, tsm, ov = tw.prune_tew(w, 0.75, 0.015, 128)
        plan = tw.TwPlan(tw.encode_cto(tsm), ov)
        x = plan.prepare(a)
        o = plan.run_tew(x, out_dtype="fp16")
        os.environ["TW_TEW_PARTS"] = "2"
        res = []
        for f in (0, 1, 2, 3, 4, 7, 15, 23, 31):
            os.environ["TW_DEBUG_FLAGS"] = str(f)
            res.append(f"flags={f}: {timed(lambda: plan.run_tew(x, out=o, out_dtype='fp16')):.2f}us")
        del os.environ["TW_DEBUG_FLAGS"], os.environ["TW_TEW_PARTS"]
        print(f"{k}x{n} K2m ablation " + " ".join(res), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "ablate":
        ablate()
    else:
        main()
