"""Paired units (TW_PAIR=1: two units of a CTA's sub-tile share every
streamed payload stage) against the regular ring on 3072 x 768 (streamed
payload, row-run layout) at several SM budgets and token counts: outputs
bit-identical, per-launch time (32-launch graphs).  Then the grouped BERT
step with each.  Diagnostic only (GPU box): python scripts/pair_probe.py
"""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2402_10876_b200 as tw  # noqa: E402
from bench import graph_us  # noqa: E402


def main():
    k, n = 3072, 768
    w = tw.round_to(tw.synthetic_matrix(0, k, n, tw.STREAM_WEIGHTS), "fp16")
    _, tsm = tw.prune_tw(w, 0.75, 128)
    plan = tw.TwPlan(tw.encode_cto(tsm), row_layout="runs")
    for m in (8192, 3001, 16384):
        a = tw.round_to(tw.synthetic_matrix(0, m, k, tw.STREAM_INPUT), "fp16")
        x = plan.prepare(torch.from_numpy(a).cuda())
        for sms in (148, 50, 24):
            plan.set_sm_budget(sms)
            res = {}
            for pair in ("0", "1"):
                os.environ["TW_PAIR"] = pair
                o = plan.run(x, out_dtype="fp16")
                torch.cuda.synchronize()
                t = graph_us(lambda i: plan.run(x, out=o, out_dtype="fp16"), 32)
                res[pair] = (o.clone(), t)
            same = torch.equal(res["0"][0], res["1"][0])
            print(f"m={m} sms={sms}: regular {res['0'][1]:.2f} us, paired {res['1'][1]:.2f} us, "
                  f"bit-identical {same}", flush=True)
        plan.set_sm_budget(0)
    os.environ.pop("TW_PAIR", None)


if __name__ == "__main__":
    main()
