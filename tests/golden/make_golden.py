"""Generate the golden vectors in tests/golden/ from the UNMODIFIED reference.

Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports tilesparse from /root/reference/pkg/src, runs its own prune /
encode / gemm functions and stores inputs and outputs.  Nothing at test or
bench time reads /root/reference; the GPU box only sees these fixtures.

Files
  small.npz   40 small TW/TEW problems (masks, CTO arrays, overlays, fp64
              gemm_cto / gemm_tew outputs) incl. tie-heavy and clamp cases
  bert.npz    BERT-base layers (768x768, 768x3072, 3072x768), fp16-rounded
              synthetic weights (seed 0): TW 0.75/G128 and TEW 0.75+0.015
              structure, fp64 outputs for the first 8 tokens, and sha256 of
              the reference's full M=8192 gemm_cto output bytes
  cfg1.npz    config 1 (1024^2 fp32, TW 0.75 G128, M=128): structure, the
              first 16 output rows and the sha256 of the full output
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import tilesparse as ref  # noqa: E402

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
from paper_2402_10876_b200.core import round_to, synthetic_matrix  # noqa: E402


def sha(arr: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()


def tw_record(prefix: str, plan, tsm, enc, store: dict, full_mask: bool = True) -> None:
    if full_mask:
        store[f"{prefix}mask"] = np.packbits(plan.element_mask.ravel())
    store[f"{prefix}mask_sha256"] = np.frombuffer(sha(plan.element_mask).encode(), dtype=np.uint8)
    store[f"{prefix}cols"] = tsm.column_mask.kept.astype(np.int32)
    store[f"{prefix}rows"] = np.concatenate([t.kept_rows.kept for t in tsm.tiles]).astype(np.int32)
    store[f"{prefix}row_counts"] = enc.row_counts.copy()
    store[f"{prefix}col_counts"] = enc.col_counts.copy()
    store[f"{prefix}row_offsets"] = enc.row_offsets.copy()
    store[f"{prefix}col_offsets"] = enc.col_offsets.copy()
    store[f"{prefix}payload_sha256"] = np.frombuffer(sha(enc.payload).encode(), dtype=np.uint8)


def small_cases():
    rng = np.random.default_rng(20260417)
    cases = []
    shapes = [(5, 4, 2), (12, 8, 4), (20, 24, 5), (33, 17, 4), (64, 48, 8), (40, 36, 8),
              (16, 16, 4), (8, 8, 2), (96, 80, 16), (128, 96, 32), (70, 130, 64), (1, 9, 4),
              (9, 1, 4), (200, 150, 128), (64, 300, 128), (300, 64, 32), (48, 64, 1),
              (17, 200, 300), (2, 2, 1), (160, 192, 128)]
    for idx, (k, n, g) in enumerate(shapes):
        for variant in range(2):
            s = float(rng.choice([0.0, 0.3, 0.5, 0.6, 0.75, 0.9]))
            delta = float(rng.choice([0.0, 0.01, 0.05, 0.1])) if s < 0.89 else 0.0
            m = int(rng.integers(1, 24))
            w = rng.normal(size=(k, n)).astype(np.float32)
            if variant == 1 and idx % 3 == 0:
                w = np.round(w, 1)          # many exact ties
            if idx == 18 and variant == 1:
                w[:] = 1.0                   # all-tie: clamp / tie-break rules
            a = rng.normal(size=(m, k)).astype(np.float32)
            cases.append((k, n, g, s, delta, m, w, a))
    return cases


def make_small() -> None:
    store, meta = {}, []
    for ci, (k, n, g, s, delta, m, w, a) in enumerate(small_cases()):
        p = f"c{ci}_"
        plan, tsm = ref.prune_tw(w, s, g)
        enc = ref.encode_cto(tsm)
        store[p + "w"] = w
        store[p + "a"] = a
        tw_record(p + "tw_", plan, tsm, enc, store)
        store[p + "tw_out"] = ref.gemm_cto(a, enc).condensed
        entry = {"k": k, "n": n, "g": g, "s": s, "delta": delta, "m": m,
                 "tw_achieved": plan.achieved_sparsity, "tw_clamps": plan.clamps,
                 "tw_params": plan.params}
        if s + delta < 1.0 and delta > 0:
            tplan, ttsm, ov = ref.prune_tew(w, s, delta, g)
            tenc = ref.encode_cto(ttsm)
            tw_record(p + "tew_", tplan, ttsm, tenc, store)
            store[p + "tew_col_ptr"] = ov.col_ptr.copy()
            store[p + "tew_row_idx"] = ov.row_idx.copy()
            store[p + "tew_values"] = ov.values.copy()
            out = ref.gemm_tew(a, ttsm, ov)
            store[p + "tew_out"] = out.condensed
            store[p + "tew_union"] = out.column_map.kept.astype(np.int32)
            entry.update({"tew": True, "tew_achieved": tplan.achieved_sparsity,
                          "tew_params": {kk: v for kk, v in tplan.params.items()}})
        else:
            entry["tew"] = False
        meta.append(entry)
    store["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(HERE / "small.npz", **store)


BERT = [(768, 768), (768, 3072), (3072, 768)]
BERT_M = 8192


def make_bert() -> None:
    store, meta = {}, []
    for li, (k, n) in enumerate(BERT):
        p = f"l{li}_"
        w = round_to(synthetic_matrix(0, k, n, 0), "fp16")
        a = round_to(synthetic_matrix(0, BERT_M, k, 1), "fp16")
        t0 = time.time()
        plan, tsm = ref.prune_tw(w, 0.75, 128)
        enc = ref.encode_cto(tsm)
        tw_record(p + "tw_", plan, tsm, enc, store, full_mask=False)
        full = ref.gemm_cto(a, enc).condensed
        store[p + "tw_out8"] = full[:8]
        tw_sha = sha(full)
        tplan, ttsm, ov = ref.prune_tew(w, 0.75, 0.015, 128)
        tenc = ref.encode_cto(ttsm)
        tw_record(p + "tew_", tplan, ttsm, tenc, store, full_mask=False)
        store[p + "tew_col_ptr"] = ov.col_ptr.astype(np.int32)
        store[p + "tew_row_idx"] = ov.row_idx.astype(np.int32)
        store[p + "tew_values"] = ov.values.copy()
        tout = ref.gemm_tew(a[:8], ttsm, ov)
        store[p + "tew_out8"] = tout.condensed
        store[p + "tew_union"] = tout.column_map.kept.astype(np.int32)
        meta.append({"k": k, "n": n, "tw_achieved": plan.achieved_sparsity,
                     "tw_clamps": plan.clamps, "tw_out_sha256": tw_sha,
                     "tew_achieved": tplan.achieved_sparsity, "tew_nnz": ov.nnz,
                     "tew_clamps": tplan.clamps, "seconds": time.time() - t0})
        print(meta[-1])
    store["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(HERE / "bert.npz", **store)


def make_cfg1() -> None:
    w = synthetic_matrix(0, 1024, 1024, 0)
    a = synthetic_matrix(0, 128, 1024, 1)
    plan, tsm = ref.prune_tw(w, 0.75, 128)
    enc = ref.encode_cto(tsm)
    store = {}
    tw_record("tw_", plan, tsm, enc, store, full_mask=False)
    out = ref.gemm_cto(a, enc).condensed
    store["out16"] = out[:16]
    meta = {"achieved": plan.achieved_sparsity, "out_sha256": sha(out),
            "flops": int(ref.report(plan, tsm, 128).sparse_flops)}
    store["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(HERE / "cfg1.npz", **store)
    print(meta)


if __name__ == "__main__":
    make_small()
    make_cfg1()
    make_bert()
