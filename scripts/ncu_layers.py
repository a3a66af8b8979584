"""ncu target (GPU box): 3 warm-up passes over the three BERT layers, then one
pass to profile (launches 9, 10, 11 of K1 -> ncu -s 9 -c 3).  Each pass uses a
different buffer set of 4 so L2 is cold-ish, as in bench.py.

    ncu --set full -k regex:tw_gemm -s 9 -c 3 -o prof python scripts/ncu_layers.py
"""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2402_10876_b200 as tw  # noqa: E402

LAYERS = [(768, 768), (768, 3072), (3072, 768)]


def main():
    torch.cuda.set_device(0)
    delta = float(os.environ.get("NCU_DELTA", "0"))
    sets = []
    for k, n in LAYERS:
        w = tw.round_to(tw.synthetic_matrix(0, k, n, 0), "fp16")
        if delta:
            _, tsm, ov = tw.prune_tew(w, 0.75, delta, 128)
        else:
            _, tsm = tw.prune_tw(w, 0.75, 128)
            ov = None
        a = tw.round_to(tw.synthetic_matrix(0, 8192, k, 1), "fp16")
        per = []
        for _ in range(4):
            plan = tw.TwPlan(tw.encode_cto(tsm), overlay=ov) if ov is not None else tw.TwPlan(
                tw.encode_cto(tsm))
            at = plan.prepare(torch.from_numpy(a).cuda())
            rows = plan.info.n_union if ov is not None else tsm.n_condensed
            out = torch.empty((rows, 8192), dtype=torch.float16, device="cuda")
            per.append((plan, at, out))
        sets.append(per)
    torch.cuda.synchronize()
    for p in range(4):
        for li in range(3):
            plan, at, out = sets[li][p]
            if delta:
                plan.run_tew(at, out=out)
            else:
                plan.run(at, out=out)
    torch.cuda.synchronize()
    print("done")


if __name__ == "__main__":
    main()
