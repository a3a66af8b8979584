"""TVW sparse (tcgen05.mma.sp) vs dense K1 on the BERT TVW layers, natural
row order, with parts switched off (TW_DEBUG_FLAGS 1: no activation loads,
4: no MMAs) and the owner / strided work split forced (TW_OWNER /
TW_STRIDED).  Diagnostic (GPU box)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2402_10876_b200 as tw  # noqa: E402
from bench import graph_us  # noqa: E402

m = 8192
for k, n in [(768, 768), (768, 3072)]:
    w = tw.round_to(tw.synthetic_matrix(0, k, n, tw.STREAM_WEIGHTS), "fp16")
    a = tw.round_to(tw.synthetic_matrix(0, m, k, tw.STREAM_INPUT), "fp16")
    _, tsm, _ = tw.prune_tvw(w, 0.75, 128)
    plan = tw.TwPlan(tw.encode_cto(tsm), row_layout="natural")
    x = plan.prepare(a)
    out = plan.run(x, out_dtype="fp16")
    print(k, n, "n_sub", plan.info.n_sub, "kp", plan.info.kp, flush=True)
    res = []
    for ns in ("0", "1", "cap256"):
        for mode in ("",):
            for fl in ("0", "36"):
                os.environ["TW_NO_SPARSE"] = "1" if ns == "1" else "0"
                os.environ["TW_SPARSE_CAP256"] = "1" if ns == "cap256" else "0"
                os.environ["TW_DEBUG_FLAGS"] = fl
                for v in ("TW_OWNER", "TW_STRIDED"):
                    os.environ[v] = "1" if v == mode else "0"
                try:
                    t = graph_us(lambda i: plan.run(x, out=out, out_dtype="fp16"), 32)
                    res.append(f"{ns} fl={fl}: {t:.2f}")
                except Exception as e:  # noqa: BLE001
                    res.append(f"sparse={1 - int(ns)} {mode or 'auto'} fl={fl}: {type(e).__name__}")
    print(k, n, " | ".join(res), flush=True)
