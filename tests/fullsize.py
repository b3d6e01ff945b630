"""Size-independent comparison helpers for the full-size parity tests
(test infrastructure only): per-task records of the reference (oracle/_ref
ref_run) and of the GPU replay (carma_task_result) in one canonical layout,
SHA-256 digests per field, IEEE bit patterns of scalars."""
from __future__ import annotations

import hashlib

import numpy as np

canon_dtype = np.dtype([
    ("first_attempt", "<f8"), ("final_dispatch", "<f8"), ("complete", "<f8"), ("first_crash", "<f8"),
    ("last_crash", "<f8"), ("executed", "<f8"), ("attempts", "<u4"), ("ooms", "<u4"), ("gpu0", "<i4"),
    ("gpu1", "<i4"),
])


def ref_tasks_canonical(tout: np.ndarray) -> np.ndarray:
    """oracle_bind.ref_task_out_dtype rows -> canon_dtype."""
    r = np.zeros(len(tout), canon_dtype)
    for f in ("first_attempt", "final_dispatch", "complete", "first_crash", "last_crash", "executed", "ooms",
              "gpu0", "gpu1"):
        r[f] = tout[f]
    r["attempts"] = tout["n_attempts"]
    return r


def gpu_tasks_canonical(tres: np.ndarray) -> np.ndarray:
    """abi.task_result_dtype rows -> canon_dtype."""
    r = np.zeros(len(tres), canon_dtype)
    for f in ("first_attempt", "final_dispatch", "complete", "first_crash", "last_crash", "executed", "attempts",
              "ooms"):
        r[f] = tres[f]
    r["gpu0"] = tres["gpu"][:, 0]
    r["gpu1"] = tres["gpu"][:, 1]
    return r


def digest_fields(rec: np.ndarray) -> dict:
    """SHA-256 of each field's contiguous little-endian bytes (row order)."""
    return {f: hashlib.sha256(np.ascontiguousarray(rec[f]).tobytes()).hexdigest() for f in rec.dtype.names}


def hex_f64(a) -> list:
    return [int(v).to_bytes(8, "big").hex() for v in np.ascontiguousarray(a, np.float64).view(np.uint64)]


def bits_of(d: dict) -> dict:
    return {k: np.float64(v).view(np.uint64).item().to_bytes(8, "big").hex() for k, v in d.items()}


def sample_records(rec: np.ndarray, stride: int) -> list:
    """Every stride-th record as {field: value} (floats as bit patterns)."""
    out = []
    for i in range(0, len(rec), stride):
        r = {"row": i}
        for f in rec.dtype.names:
            v = rec[f][i]
            r[f] = np.float64(v).view(np.uint64).item().to_bytes(8, "big").hex() if rec.dtype[f].kind == "f" \
                else int(v)
        out.append(r)
    return out


def first_mismatch(a: np.ndarray, b: np.ndarray):
    """(field, row) of the first differing value (bitwise for floats), or None."""
    for f in a.dtype.names:
        x, y = np.ascontiguousarray(a[f]), np.ascontiguousarray(b[f])
        if x.dtype.kind == "f":
            x, y = x.view(np.uint64), y.view(np.uint64)
        bad = np.nonzero(x != y)[0]
        if len(bad):
            return f, int(bad[0])
    return None
