"""Per-stage clock64 timeline of K1 (diagnostics; GPU box).

    python scripts/ktrace.py [--layer 0|1|2] [--mode 1] [--flags 0]
"""
import argparse
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2402_10876_b200 as tw  # noqa: E402
from paper_2402_10876_b200 import _native  # noqa: E402

LAYERS = [(768, 768), (768, 3072), (3072, 768)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layer", type=int, default=0)
    ap.add_argument("--mode", default="1")
    ap.add_argument("--flags", default="0")
    ap.add_argument("--m", type=int, default=8192)
    ap.add_argument("--shape", default="", help="KxN instead of a BERT layer (e.g. 1024x1024)")
    args = ap.parse_args()
    os.environ["TW_GATHER"] = args.mode
    os.environ["TW_DEBUG_FLAGS"] = args.flags
    k, n = (tuple(int(v) for v in args.shape.split("x")) if args.shape else LAYERS[args.layer])
    w = tw.round_to(tw.synthetic_matrix(0, k, n, 0), "fp16")
    _, tsm = tw.prune_tw(w, 0.75, 128)
    plan = tw.TwPlan(tw.encode_cto(tsm), row_layout=os.environ.get('TW_ROW_LAYOUT', 'runs'))
    a = tw.round_to(tw.synthetic_matrix(0, args.m, k, 1), "fp16")
    at = plan.prepare(torch.from_numpy(a).cuda())
    out = torch.empty((tsm.n_condensed, args.m), dtype=torch.float16, device="cuda")
    for _ in range(3):
        plan.run(at, out=out)
    buf = torch.zeros((148, 4096), dtype=torch.int64, device="cuda")
    lib = _native.load_library()
    lib.tw_debug_set_trace(buf.data_ptr())
    torch.cuda.synchronize()
    plan.run(at, out=out)
    torch.cuda.synchronize()
    lib.tw_debug_set_trace(None)
    t = buf.cpu().numpy()
    print(f"layer {k}x{n} mode={args.mode} flags={args.flags}")
    full_ts, epi = [], []
    ends = []
    first_active = int(np.argmax(t[:, 1024] != 0))
    for c in range(148):
        t0 = t[c, 3072]
        if t0 == 0:
            continue
        ful = t[c, 1024:2048]
        ns = int(np.count_nonzero(ful))
        e = t[c, 2048:2048 + 512].reshape(-1, 2)
        e = e[e[:, 0] > 0]
        if ns:
            full_ts.append(ful[ns - 1] - t0)
        if len(e):
            ends.append(e[-1, 1] - t0)
            epi.extend((e[:, 1] - e[:, 0]).tolist())
        if c == first_active:
            iss = np.where(t[c, 0:ns] > 0, t[c, 0:ns] - t0, 0)
            f = ful[:ns] - t0
            print(f"  cta {c} issue/full/lat: " + " ".join(f"{int(a)}/{int(b)}/{int(b - a)}" for a, b in zip(iss[:16], f[:16])))
        if c < 4 or c in (74, 147):
            f = ful[:ns] - t0
            print(f" cta {c}: stages {ns}, full at {f[:3].tolist()}..{f[-2:].tolist()}, "
                  "epi " + ", ".join(f"[{a0 - t0}, {a1 - t0}]" for a0, a1 in e))
    q = lambda v: np.percentile(v, [10, 50, 90, 100]).astype(int).tolist() if len(v) else []
    print(" last-full p10/50/90/max", q(full_ts))
    g0 = t[:, 3074][t[:, 3074] > 0]
    g1 = t[:, 3075][t[:, 3075] > 0]
    if len(g0) and len(g1):
        print(f" globaltimer: CTA starts spread {int(g0.max() - g0.min())} ns, "
              f"first start -> last epilogue end {int(g1.max() - g0.min())} ns, "
              f"median CTA body {int(np.median(g1 - g0[:len(g1)]))} ns")
    print(" cta end (last epilogue) p10/50/90/max", q(ends))
    # per-CTA summary: stages, boxes (run path), last full, end
    rows = []
    for c in range(148):
        t0 = t[c, 3072]
        if t0 == 0:
            continue
        ful = t[c, 1024:2048]
        ns = int(np.count_nonzero(ful))
        e = t[c, 2048:2048 + 512].reshape(-1, 2)
        e = e[e[:, 0] > 0]
        rows.append((c, ns, int(t[c, 3076]), int(ful[ns - 1] - t0) if ns else 0,
                     int(e[-1, 1] - t0) if len(e) else 0, int(ful[0] - t0) if ns else 0))
    print(" per-CTA cta:stages/boxes/first/lastfull/end")
    for i in range(0, len(rows), 6):
        print("  " + "  ".join(f"{c}:{ns}/{nb}/{f0}/{lf}/{en}" for c, ns, nb, lf, en, f0 in rows[i:i + 6]))
    print(" epilogue per segment p10/50/90/max", q(epi))


if __name__ == "__main__":
    main()
