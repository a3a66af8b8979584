"""Probe (GPU box): grouped BERT step time over a grid of SM budgets."""
import itertools
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2402_10876_b200 as tw  # noqa: E402
from scripts.group_probe import LAYERS, R, graph_time  # noqa: E402


def main():
    m = 8192
    encs = []
    for k, n in LAYERS:
        w = tw.round_to(tw.synthetic_matrix(0, k, n, 0), "fp16")
        encs.append(tw.encode_cto(tw.prune_tw(w, 0.75, 128)[1]))
    layout = sys.argv[1] if len(sys.argv) > 1 else "runs"
    sets = []
    for r in range(R):
        plans = [tw.TwPlan(e, row_layout=layout) for e in encs]
        xs = [p.prepare(torch.from_numpy(tw.round_to(tw.synthetic_matrix(r, m, k, 1), "fp16")).cuda())
              for p, (k, n) in zip(plans, LAYERS)]
        outs = [torch.empty((p.info.n_condensed, m), dtype=torch.float16, device="cuda") for p in plans]
        sets.append((plans, xs, outs))
    streams = [torch.cuda.Stream() for _ in range(3)]
    res = []
    for b0, b1 in itertools.product([12, 15, 18, 21], [70, 76, 82, 88]):
        b2 = 148 - b0 - b1
        for plans, _, _ in sets:
            for p, b in zip(plans, (b0, b1, b2)):
                p.set_sm_budget(b)

        def grp(i):
            plans, xs, outs = sets[i]
            cur = torch.cuda.current_stream()
            ev = torch.cuda.Event()
            ev.record(cur)
            js = []
            for s, p, x, o in zip(streams, plans, xs, outs):
                s.wait_event(ev)
                with torch.cuda.stream(s):
                    p.run(x, out=o, stream=s)
                e = torch.cuda.Event()
                e.record(s)
                js.append(e)
            for e in js:
                cur.wait_event(e)

        t = graph_time(grp)
        res.append((t, b0, b1, b2))
        print(f"budgets {b0:3d} {b1:3d} {b2:3d}: {t:.1f} us", flush=True)
    res.sort()
    print("best", res[:3])


if __name__ == "__main__":
    main()
