"""Per-CTA start / last-epilogue times of the one-launch grouped BERT step
(tw_gemm_group; one trace buffer, slot = global CTA index), 4 steps in a
CUDA graph.  Diagnostic (GPU box)."""
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
        p = tw.TwPlan(tw.encode_cto(tw.prune_tw(w, 0.75, 128)[1]), row_layout="runs")
        plans.append(p)
        xs.append(p.prepare(torch.from_numpy(tw.round_to(tw.synthetic_matrix(0, m, k, 1), "fp16")).cuda()))
        outs.append(torch.empty((p.info.n_condensed, m), dtype=torch.float16, device="cuda"))
    grp = tw.TwPlanGroup(plans, m)
    buf = torch.zeros(160 * 4096, dtype=torch.int64, device="cuda")
    lib.tw_debug_set_trace(buf.data_ptr())
    g = capture_graph(lambda: [grp.run(xs, outs, out_dtype="fp16") for _ in range(4)])
    lib.tw_debug_set_trace(None)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"{e0.elapsed_time(e1) / 20 * 1e3:.1f} us per step (traced), budgets {grp.budgets}")
    buf.zero_()
    g.replay()
    torch.cuda.synchronize()
    t = buf.view(160, 4096).cpu()
    start, end = t[:, 3074], t[:, 3075]
    t0 = int(start[start > 0].min())
    c0 = 0
    for (k, n), b in zip(LAYERS, grp.budgets):
        s, e = start[c0:c0 + b], end[c0:c0 + b]
        live = s > 0
        s, e = s[live], e[live & (e > 0)]
        print(f"{k}x{n}: CTAs {int(live.sum())}: start {(int(s.min()) - t0) / 1e3:6.2f}..{(int(s.max()) - t0) / 1e3:6.2f} us, "
              f"done {(int(e.min()) - t0) / 1e3:6.2f}..{(int(e.max()) - t0) / 1e3:6.2f} us", flush=True)
        # clock64 phases per CTA (cycles from the CTA's prologue end)
        ph = []
        for c in range(c0, c0 + b):
            tc = t[c]
            if tc[3072] == 0:
                continue
            ful = tc[1024:2048]
            ns = int((ful != 0).sum())
            ep = tc[2048:2560].view(-1, 2)
            ep = ep[ep[:, 0] > 0]
            if ns < 2 or len(ep) == 0:
                continue
            first, last = int(ful[0] - tc[3072]), int(ful[ns - 1] - tc[3072])
            endc = int(ep[-1, 1] - tc[3072])
            ph.append((first, (last - first) / (ns - 1), endc - last, ns, len(ep)))
        if ph:
            import statistics as st
            cols = list(zip(*ph))
            print("    first-full {:.0f} | cycles/stage {:.0f} | last-full->end {:.0f} | stages {:.0f} | units {:.1f}"
                  .format(*(st.median(v) for v in cols)), flush=True)
        c0 += b


if __name__ == "__main__":
    main()
