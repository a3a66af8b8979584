"""Probe (GPU box): the BERT step as 3 sequential K1 launches vs a
TwPlanGroup (SM shares, concurrent streams), and cuBLAS both ways.

    python scripts/group_probe.py [--m 8192] [--layout runs|natural]
"""
import argparse
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2402_10876_b200 as tw  # noqa: E402

LAYERS = [(768, 768), (768, 3072), (3072, 768)]
R = 4


def graph_time(fn, steps=32):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for i in range(R):
            fn(i)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for i in range(steps):
                fn(i % R)
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(7):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / steps)
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=8192)
    ap.add_argument("--layout", default="runs")
    ap.add_argument("--sms", type=int, default=0)
    args = ap.parse_args()
    m = args.m
    torch.cuda.set_device(0)
    encs, ws = [], []
    for k, n in LAYERS:
        w = tw.round_to(tw.synthetic_matrix(0, k, n, 0), "fp16")
        _, tsm = tw.prune_tw(w, 0.75, 128)
        encs.append(tw.encode_cto(tsm))
        ws.append(w)
    sets = []
    for r in range(R):
        plans = [tw.TwPlan(e, row_layout=args.layout) for e in encs]
        xs = [p.prepare(torch.from_numpy(tw.round_to(tw.synthetic_matrix(r, m, k, 1), "fp16")).cuda())
              for p, (k, n) in zip(plans, LAYERS)]
        outs = [torch.empty((p.info.n_condensed, m), dtype=torch.float16, device="cuda") for p in plans]
        sets.append((plans, xs, outs))
    flops = sum(sets[0][0][i].flops(m) for i in range(3))

    def seq(i):
        plans, xs, outs = sets[i]
        for p, x, o in zip(plans, xs, outs):
            p.run(x, out=o)

    t_seq = graph_time(seq)
    ref = [o.clone() for o in sets[0][2]]
    groups = [tw.TwPlanGroup(sets[r][0], m, sms=args.sms or None) for r in range(R)]
    print("budgets", groups[0].budgets, "stage_work", [int(p.info.stage_work) for p in sets[0][0]])

    def grp(i):
        plans, xs, outs = sets[i]
        groups[i].run(xs, outs)

    t_grp = graph_time(grp)
    grp(0)
    torch.cuda.synchronize()
    same = all(torch.equal(a, b) for a, b in zip(ref, sets[0][2]))
    # per-layer times on the budgets (alone)
    alone = []
    for li in range(3):
        def one(i, li=li):
            plans, xs, outs = sets[i]
            plans[li].run(xs[li], out=outs[li])
        alone.append(graph_time(one))
    # cuBLAS
    dense = []
    for r in range(R):
        row = []
        for (k, n), w in zip(LAYERS, ws):
            wt = torch.from_numpy(np.ascontiguousarray(w.T)).cuda().half()
            at = torch.randn((k, m), device="cuda", dtype=torch.float16)
            row.append((wt, at, torch.empty((n, m), device="cuda", dtype=torch.float16)))
        dense.append(row)

    def dseq(i):
        for wt, at, o in dense[i]:
            torch.matmul(wt, at, out=o)

    streams = [torch.cuda.Stream() for _ in range(3)]

    def dgrp(i):
        cur = torch.cuda.current_stream()
        ev = torch.cuda.Event()
        ev.record(cur)
        joins = []
        for s, (wt, at, o) in zip(streams, dense[i]):
            s.wait_event(ev)
            with torch.cuda.stream(s):
                torch.matmul(wt, at, out=o)
            e = torch.cuda.Event()
            e.record(s)
            joins.append(e)
        for e in joins:
            cur.wait_event(e)

    t_dseq = graph_time(dseq)
    t_dgrp = graph_time(dgrp)
    print(f"ours: sequential {t_seq:.1f} us, grouped {t_grp:.1f} us (bit-identical {same}); "
          f"alone on budget {[round(a, 1) for a in alone]}")
    print(f"cuBLAS: sequential {t_dseq:.1f} us, 3 streams {t_dgrp:.1f} us")
    print(f"speedup: seq/seq {t_dseq / t_seq:.2f}x, grouped/seq-cublas {t_dseq / t_grp:.2f}x, "
          f"grouped/grouped-cublas {t_dgrp / t_grp:.2f}x; grouped {flops / t_grp / 1e6:.0f} TFLOP/s")




def soak_ab():
    """Sustained-load A/B: grouped vs sequential steps alternated after a
    2 s soak (power-capped clocks), 5 rounds each."""
    import time
    m = 8192
    encs = []
    for k, n in LAYERS:
        w = tw.round_to(tw.synthetic_matrix(0, k, n, 0), "fp16")
        encs.append(tw.encode_cto(tw.prune_tw(w, 0.75, 128)[1]))
    sets = []
    for r in range(R):
        plans = [tw.TwPlan(e, row_layout="runs") for e in encs]
        xs = [p.prepare(torch.from_numpy(tw.round_to(tw.synthetic_matrix(r, m, k, 1), "fp16")).cuda())
              for p, (k, n) in zip(plans, LAYERS)]
        outs = [torch.empty((p.info.n_condensed, m), dtype=torch.float16, device="cuda") for p in plans]
        sets.append((plans, xs, outs))
    groups = [tw.TwPlanGroup(sets[r][0], m) for r in range(R)]

    def seq(i):
        for p, x, o in zip(*sets[i]):
            p.run(x, out=o)

    def grp(i):
        groups[i].run(sets[i][1], sets[i][2])

    def cap(fn):
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for i in range(R):
                fn(i)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for i in range(64):
                    fn(i % R)
        torch.cuda.current_stream().wait_stream(s)
        return g

    # budgets are plan state: grouped graph captured with budgets set, the
    # sequential graph with the same plans at full budget (set per replay)
    gg = cap(grp)
    for g in groups:
        g.release()
    gs = cap(seq)
    for g, r in zip(groups, range(R)):
        for p, b in zip(sets[r][0], g.budgets):
            p.set_sm_budget(b)
    t0 = time.time()
    while time.time() - t0 < 2.0:
        gg.replay()
    torch.cuda.synchronize()
    res = {"grouped": [], "sequential": []}
    for _ in range(5):
        for name, g in (("grouped", gg), ("sequential", gs)):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(8):
                g.replay()
            e1.record()
            torch.cuda.synchronize()
            res[name].append(e0.elapsed_time(e1) * 1e3 / (8 * 64))
    print("sustained A/B us per step:", {k: [round(v, 1) for v in vs] for k, vs in res.items()})


if __name__ == "__main__":
    if "--soak" in sys.argv:
        soak_ab()
    else:
        main()
