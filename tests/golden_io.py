"""Loaders for the reference-generated golden documents (tests/golden/)."""

from __future__ import annotations

import functools
import gzip
import json
import math
import os

import numpy as np

from paper_1801_08058_b200.serialize import document_to_function, document_to_tensor

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@functools.lru_cache(maxsize=None)
def load(name: str):
    with gzip.open(os.path.join(GOLDEN, name), "rt") as fh:
        return json.load(fh)


def fn_of(doc):
    return document_to_function(doc)


def tensor_of(doc):
    return document_to_tensor(doc)


def logical(doc) -> np.ndarray:
    return document_to_tensor(doc).to_numpy()


def same_bits(a: np.ndarray, b: np.ndarray) -> bool:
    """Bit equality with every NaN treated as equal (payloads differ by platform)."""
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    if a.shape != b.shape or a.dtype != b.dtype:
        return False
    if a.dtype.kind == "f":
        na, nb = np.isnan(a), np.isnan(b)
        if not np.array_equal(na, nb):
            return False
        bits = np.uint32 if a.dtype == np.float32 else np.uint64
        return bool(np.array_equal(a[~na].view(bits), b[~nb].view(bits)))
    return bool(np.array_equal(a, b))


def max_abs_diff(a: np.ndarray, b: np.ndarray) -> float:
    """Reference `_graphgen.max_abs_difference` semantics (NaN == NaN)."""
    a = np.asarray(a, dtype=np.float64) if a.dtype.kind == "f" else a
    b = np.asarray(b, dtype=np.float64) if b.dtype.kind == "f" else b
    if a.dtype.kind != "f":
        return 0.0 if np.array_equal(a, b) else math.inf
    both_nan = np.isnan(a) & np.isnan(b)
    with np.errstate(invalid="ignore"):
        d = np.where(both_nan | (a == b), 0.0, np.abs(a - b))
    d = np.where(np.isnan(d), math.inf, d)
    return float(d.max()) if d.size else 0.0


def normwise(a: np.ndarray, ref: np.ndarray) -> float:
    """max|a - ref| / max|ref| (SURVEY.md §8(c) tolerance for Sum/Dot/Conv)."""
    a = np.asarray(a, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    if ref.size == 0:
        return 0.0
    scale = max(float(np.max(np.abs(ref))), 1e-30)
    return float(np.max(np.abs(a - ref))) / scale
