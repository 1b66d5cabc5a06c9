"""Bit-exact array fingerprints shared by the golden generator and the tests."""

import hashlib

import numpy as np


def digest(a) -> dict:
    a = np.ascontiguousarray(a)
    h = hashlib.sha256()
    h.update(str(a.dtype.str).encode())
    h.update(str(tuple(a.shape)).encode())
    h.update(a.tobytes())
    return {"sha256": h.hexdigest(), "dtype": a.dtype.str, "shape": list(a.shape)}


def same(a, d: dict) -> bool:
    return digest(a)["sha256"] == d["sha256"]
