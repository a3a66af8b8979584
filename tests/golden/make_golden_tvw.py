"""Golden vectors for the TVW pattern (prune_tvw -> encode_cto -> gemm) from the
UNMODIFIED reference.  Run in the build container (the only place
/root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_tvw.py

tvw.npz
  c{i}_*      30 small problems (ragged heights for the tail vectors, ties,
              targets 0.5-0.95, g 1-32): inputs, element mask, kept rows,
              payload bytes, 2:4 offsets, plan params, fp64 gemm_tile_sparse
              output for a small activation matrix
  bert_*      BERT 768x768 fp16-rounded synthetic weights (seed 0), TVW 0.75
              G128: mask / payload / offsets sha256, CTO arrays, the first 8
              output rows of gemm_cto at M=8192 and the sha256 of the full
              fp64 output
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import tilesparse as ref  # noqa: E402

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
from paper_2402_10876_b200.core import round_to, synthetic_matrix  # noqa: E402


def sha(arr) -> np.ndarray:
    return np.frombuffer(hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest().encode(),
                         dtype=np.uint8)


def record(prefix, plan, tsm, meta, store):
    store[prefix + "mask"] = np.packbits(plan.element_mask.ravel())
    store[prefix + "cols"] = tsm.column_mask.kept.astype(np.int32)
    store[prefix + "rows"] = np.concatenate([t.kept_rows.kept for t in tsm.tiles]).astype(np.int32)
    store[prefix + "payload"] = np.concatenate([t.payload.ravel() for t in tsm.tiles])
    store[prefix + "offsets"] = np.concatenate([o.ravel() for o in meta.kept_offsets])
    store[prefix + "params"] = np.frombuffer(json.dumps(
        {"params": plan.params, "clamps": plan.clamps,
         "achieved": plan.achieved_sparsity}, sort_keys=True).encode(), dtype=np.uint8)


def main():
    rng = np.random.default_rng(20261017)
    store = {}
    meta_rows = []
    for i in range(30):
        k = int(rng.integers(5, 90))
        n = int(rng.integers(3, 70))
        g = int(rng.choice([1, 2, 4, 8, 16, 32]))
        s = float(rng.choice([0.5, 0.55, 0.625, 0.7, 0.75, 0.8, 0.9, 0.95]))
        w = rng.standard_normal((k, n)).astype(np.float32)
        if i % 4 == 0:
            w = np.round(w * 2) / 2          # many equal magnitudes: tie-breaks
        a = rng.standard_normal((int(rng.integers(1, 24)), k)).astype(np.float32)
        plan, tsm, meta = ref.prune_tvw(w, s, g)
        out = ref.gemm_tile_sparse(a, tsm)
        p = f"c{i}_"
        store[p + "w"] = w
        store[p + "a"] = a
        store[p + "out"] = out.condensed
        record(p, plan, tsm, meta, store)
        meta_rows.append({"k": k, "n": n, "g": g, "s": s})
    w = round_to(synthetic_matrix(0, 768, 768, 0), "fp16")
    a = round_to(synthetic_matrix(0, 8192, 768, 1), "fp16")
    plan, tsm, meta = ref.prune_tvw(w, 0.75, 128)
    enc = ref.encode_cto(tsm)
    out = ref.gemm_cto(a, enc).condensed
    store["bert_mask_sha256"] = sha(plan.element_mask)
    store["bert_payload_sha256"] = sha(enc.payload)
    store["bert_offsets_sha256"] = sha(np.concatenate([o.ravel() for o in meta.kept_offsets]))
    store["bert_row_offsets"] = enc.row_offsets.copy()
    store["bert_col_offsets"] = enc.col_offsets.copy()
    store["bert_row_counts"] = enc.row_counts.copy()
    store["bert_col_counts"] = enc.col_counts.copy()
    store["bert_out8"] = out[:8].copy()
    store["bert_out_sha256"] = sha(out)
    store["meta"] = np.frombuffer(json.dumps(meta_rows).encode(), dtype=np.uint8)
    np.savez_compressed(HERE / "tvw.npz", **store)
    print("wrote", HERE / "tvw.npz")


if __name__ == "__main__":
    main()
