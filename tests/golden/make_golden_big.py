"""Golden fingerprints of the reference's pruning at the large BASELINE sizes
(bit-exact pruning pinned at 16384^2, and the VGG-16 shapes of
configs[3]).

Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_big.py

It imports the UNMODIFIED tilesparse from /root/reference/pkg/src, prunes and
encodes with the reference's own functions and stores sha256 fingerprints
(the arrays themselves are too large to commit) of the element mask, the
kept columns, every tile's kept rows and the CTO arrays, plus the small
per-tile count vectors in full.  tests/test_host_parity.py recomputes them
with this repo's host restatement.
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

VGG = {"conv1_2": (576, 64), "conv2_1": (576, 128), "conv3_2": (2304, 256),
       "conv4_2": (4608, 512), "conv5_1": (4608, 512)}


def sha(arr) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()


def fingerprint(plan, tsm, enc, ov=None) -> dict:
    d = {"mask": sha(plan.element_mask),
         "cols": sha(tsm.column_mask.kept.astype(np.int64)),
         "rows": sha(np.concatenate([t.kept_rows.kept for t in tsm.tiles]).astype(np.int64)),
         "row_counts": enc.row_counts.astype(int).tolist(),
         "col_counts": enc.col_counts.astype(int).tolist(),
         "row_offsets": sha(enc.row_offsets), "col_offsets": sha(enc.col_offsets),
         "payload": sha(enc.payload), "achieved": float(plan.achieved_sparsity)}
    if ov is not None:
        d.update({"ov_col_ptr": sha(ov.col_ptr.astype(np.int64)),
                  "ov_row_idx": sha(ov.row_idx.astype(np.int64)),
                  "ov_values": sha(ov.values.astype(np.float32)), "ov_nnz": int(ov.nnz)})
    return d


def main() -> None:
    out = {}
    t0 = time.time()
    w = round_to(synthetic_matrix(0, 16384, 16384, 0), "fp16")
    plan, tsm = ref.prune_tw(w, 0.75, 128)
    out["big_tw"] = fingerprint(plan, tsm, ref.encode_cto(tsm))
    print(f"16384^2 TW: {time.time() - t0:.1f} s", flush=True)
    del w, plan, tsm
    w = round_to(synthetic_matrix(0, 4096, 4096, 0), "fp16")
    plan, tsm, ov = ref.prune_tew(w, 0.75, 0.015, 128)
    out["tew_4096"] = fingerprint(plan, tsm, ref.encode_cto(tsm), ov)
    print(f"4096^2 TEW: {time.time() - t0:.1f} s", flush=True)
    for name, (k, n) in VGG.items():
        w = round_to(synthetic_matrix(0, k, n, 0), "fp16")
        for s in (0.5, 0.7, 0.9):
            for g in (64, 128, 256):
                plan, tsm = ref.prune_tw(w, s, g)
                out[f"{name}_s{s}_g{g}"] = fingerprint(plan, tsm, ref.encode_cto(tsm))
    print(f"VGG: {time.time() - t0:.1f} s", flush=True)
    (HERE / "big.json").write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()
