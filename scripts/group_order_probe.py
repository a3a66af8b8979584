"""Fused grouped BERT step (one launch) with the layers in different orders
inside the launch (CTA order decides which layer gets freed SMs first under
programmatic dependent launch), 4 rotating sets (> 2 x L2), budgets tuned
per order.  Diagnostic (GPU box)."""
import itertools
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2402_10876_b200 as tw  # noqa: E402
from bench import capture_graph  # noqa: E402

LAYERS = [(768, 768), (768, 3072), (3072, 768)]
R = 4


def main():
    m = 8192
    sets = []
    for r in range(R):
        plans, xs, outs = [], [], []
        for k, n in LAYERS:
            w = tw.round_to(tw.synthetic_matrix(r, k, n, 0), "fp16")
            p = tw.TwPlan(tw.encode_cto(tw.prune_tw(w, 0.75, 128)[1]), row_layout="runs")
            plans.append(p)
            xs.append(p.prepare(torch.from_numpy(tw.round_to(tw.synthetic_matrix(r, m, k, 1), "fp16")).cuda()))
            outs.append(torch.empty((p.info.n_condensed, m), dtype=torch.float16, device="cuda"))
        sets.append((plans, xs, outs))
    for order in itertools.permutations(range(3)):
        groups = [tw.TwPlanGroup([sets[r][0][i] for i in order], m) for r in range(R)]

        def rot():
            for r in range(R):
                groups[r].run([sets[r][1][i] for i in order], [sets[r][2][i] for i in order],
                              out_dtype="fp16")

        def time_fn():
            g = capture_graph(rot)
            for _ in range(2):
                g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(6):
                g.replay()
            e1.record()
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / 6 / R * 1e3

        t_model = time_fn()
        best, t_best, _ = tw.tune_budgets(groups, time_fn)
        print(f"order {[f'{LAYERS[i][0]}x{LAYERS[i][1]}' for i in order]}: model {groups[0].budgets if False else ''}"
              f"{t_model:.1f} us, tuned {best} {t_best:.1f} us", flush=True)
        for g in groups:
            g.release()


if __name__ == "__main__":
    main()
