"""Shared fixtures loaders for the parity tests (test infrastructure)."""

from __future__ import annotations

import hashlib
import json
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


def sha(arr) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()


def load_npz(name: str):
    z = np.load(GOLDEN / name)
    meta = json.loads(bytes(z["meta"]).decode())
    return z, meta


def golden_str(z, key: str) -> str:
    return bytes(z[key]).decode()


def tiles_from_record(z, prefix: str):
    """Per-tile kept rows (list of int64 arrays) from a golden record."""
    counts = z[prefix + "row_counts"].astype(np.int64)
    rows = z[prefix + "rows"].astype(np.int64)
    out, pos = [], 0
    for c in counts:
        out.append(rows[pos:pos + c])
        pos += c
    return out
