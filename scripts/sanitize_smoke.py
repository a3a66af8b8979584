"""Small TW + TEW + transpose run for compute-sanitizer (GPU box):

    compute-sanitizer --tool memcheck|racecheck|synccheck python scripts/sanitize_smoke.py

Covers the resident (K' <= 448) and streamed K1 kernels in owner and strided
modes, ragged M / widths, 16-bit and fp32 outputs, K2 and both K4 paths.
"""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2402_10876_b200 as tw  # noqa: E402


def main():
    rng = np.random.default_rng(0)
    for (k, n, m, s, g) in [(256, 384, 300, 0.75, 128), (1024, 512, 200, 0.5, 128),
                            (96, 80, 37, 0.3, 16)]:
        w = tw.round_to(rng.standard_normal((k, n)).astype(np.float32), "fp16")
        a = tw.round_to(rng.standard_normal((m, k)).astype(np.float32), "fp16")
        _, tsm = tw.prune_tw(w, s, g)
        for od in ("fp32", "fp16"):
            tw.gemm_tile_sparse(a, tsm, out_dtype=od)
        os.environ["TW_STRIDED"] = "1"
        tw.TwPlan(tw.encode_cto(tsm)).run(tw.prepare_activations(a))
        del os.environ["TW_STRIDED"]
        _, ttsm, ov = tw.prune_tew(w, s, 0.02, g)
        tw.gemm_tew(a, ttsm, ov, out_dtype="fp16")
        tw.prepare_activations(torch.from_numpy(a).cuda().half())
    torch.cuda.synchronize()
    print("sanitize smoke done")


if __name__ == "__main__":
    main()
