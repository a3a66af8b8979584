"""768 x 3072 (12 tiles) K1 at several SM budgets: the cp.async gather on the
single row order against the TMA row-run path on G permuted copies of A^T
(TW_RUN_COPIES at plan creation), and the whole grouped BERT step with each.
Diagnostic only (GPU box): python scripts/copies_probe.py
"""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2402_10876_b200 as tw  # noqa: E402
from bench import graph_us  # noqa: E402

M = 8192


def layer(k, n, copies):
    os.environ["TW_RUN_COPIES"] = str(copies)
    w = tw.round_to(tw.synthetic_matrix(0, k, n, tw.STREAM_WEIGHTS), "fp16")
    _, tsm = tw.prune_tw(w, 0.75, 128)
    plan = tw.TwPlan(tw.encode_cto(tsm), row_layout="runs")
    a = tw.round_to(tw.synthetic_matrix(0, M, k, tw.STREAM_INPUT), "fp16")
    x = plan.prepare(torch.from_numpy(a).cuda())
    o = plan.run(x, out_dtype="fp16")
    del os.environ["TW_RUN_COPIES"]
    return plan, x, o


def main():
    for copies in (1, 2, 3, 4):
        plan, x, o = layer(768, 3072, copies)
        ref = o.clone()
        line = [f"copies={copies} runs={int(plan.uses_row_runs)}"]
        for sms in (148, 100, 82, 70):
            plan.set_sm_budget(sms)
            plan.run(x, out=o, out_dtype="fp16")
            torch.cuda.synchronize()
            assert torch.equal(o, ref)
            line.append(f"{sms} SMs {graph_us(lambda i: plan.run(x, out=o, out_dtype='fp16'), 32):.2f} us")
        plan.set_sm_budget(0)
        print(" | ".join(line), flush=True)
        plans, xs, outs = [], [], []
        for (k, n) in [(768, 768), (768, 3072), (3072, 768)]:
            p, xx, oo = layer(k, n, copies if n == 3072 else 1)
            plans.append(p)
            xs.append(xx)
            outs.append(oo)
        g = tw.TwPlanGroup(plans, M)
        step = graph_us(lambda i: g.run(xs, outs, out_dtype="fp16"), 16)
        def timed():
            return graph_us(lambda i: g.run(xs, outs, out_dtype="fp16"), 16)
        budgets, t, _ = tw.tune_budgets([g], timed)
        print(f"   grouped step (warm L2): default shares {step:.2f} us; tuned {budgets} "
              f"{t:.2f} us", flush=True)




def shares():
    """Each BERT layer alone at the grouped step's tuned SM shares."""
    for copies, budgets in ((1, (16, 84, 48)), (3, (21, 77, 50))):
        line = [f"copies={copies}"]
        for (k, n), b in zip([(768, 768), (768, 3072), (3072, 768)], budgets):
            p, xx, oo = layer(k, n, copies if n == 3072 else 1)
            p.set_sm_budget(b)
            line.append(f"{k}x{n}@{b}: {graph_us(lambda i: p.run(xx, out=oo, out_dtype='fp16'), 32):.2f} us")
        print(" | ".join(line), flush=True)


if __name__ == "__main__":
    shares() if sys.argv[1:] == ["shares"] else main()
