"""When does each layer of the grouped BERT step start and finish?  Each
layer's K1 launch gets its own trace buffer (per-CTA globaltimer at start,
slot 3074, and after the last epilogue, slot 3075); the group is launched
like TwPlanGroup.run (fork / join over 3 streams) inside a CUDA graph,
several steps back to back.  Diagnostic (GPU box)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2402_10876_b200 as tw  # noqa: E402
from paper_2402_10876_b200 import _native  # noqa: E402
from bench import capture_graph  # noqa: E402

LAYERS = [(768, 768), (768, 3072), (3072, 768)]


def main():
    m = 8192
    lib = _native.load_library()
    plans, xs, outs = [], [], []
    for k, n in LAYERS:
        w = tw.round_to(tw.synthetic_matrix(0, k, n, 0), "fp16")
        p = tw.TwPlan(tw.encode_cto(tw.prune_tw(w, 0.75, 128)[1]))
        plans.append(p)
        xs.append(p.prepare(torch.from_numpy(tw.round_to(tw.synthetic_matrix(0, m, k, 1), "fp16")).cuda()))
        outs.append(torch.empty((p.info.n_condensed, m), dtype=torch.float16, device="cuda"))
    grp = tw.TwPlanGroup(plans, m)
    bufs = [torch.zeros(148 * 4096, dtype=torch.int64, device="cuda") for _ in plans]
    streams = grp.streams

    def step():
        cur = torch.cuda.current_stream()
        fork = torch.cuda.Event()
        fork.record(cur)
        joins = []
        for p, s, x, o, b in zip(plans, streams, xs, outs, bufs):
            s.wait_event(fork)
            with torch.cuda.stream(s):
                lib.tw_debug_set_trace(b.data_ptr())
                p.run(x, out=o, stream=s)
            e = torch.cuda.Event()
            e.record(s)
            joins.append(e)
        for e in joins:
            cur.wait_event(e)
        lib.tw_debug_set_trace(None)

    import os
    for gran in os.environ.get("GRANS", "64").split(","):
        os.environ["TW_GRAN"] = gran
        print(f"TW_GRAN={gran}", flush=True)
        trace_once(step, bufs, plans, grp)


def trace_once(step, bufs, plans, grp):
    g = capture_graph(lambda: [step() for _ in range(4)])
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    for b in bufs:
        b.zero_()
    g.replay()  # the traces hold the 4th step of this replay (last writer wins)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"  {e0.elapsed_time(e1) / 20 * 1e3:.1f} us per step (traced)", flush=True)
    for b in bufs:
        b.zero_()
    g.replay()
    torch.cuda.synchronize()
    t0 = None
    rows = []
    for (k, n), p, b, budget in zip(LAYERS, plans, bufs, grp.budgets):
        t = b.view(148, 4096).cpu()
        start, end = t[:, 3074], t[:, 3075]
        live = start > 0
        s, e = start[live], end[live & (end > 0)]
        rows.append((f"{k}x{n}", budget, int(live.sum()), int(s.min()), int(s.max()), int(e.min()), int(e.max())))
        t0 = int(s.min()) if t0 is None else min(t0, int(s.min()))
    for name, budget, ctas, s0, s1, e0, e1 in rows:
        print(f"{name}: budget {budget}, CTAs {ctas}: start {(s0 - t0) / 1e3:6.2f}..{(s1 - t0) / 1e3:6.2f} us, "
              f"last epilogue done {(e0 - t0) / 1e3:6.2f}..{(e1 - t0) / 1e3:6.2f} us", flush=True)


if __name__ == "__main__":
    main()
