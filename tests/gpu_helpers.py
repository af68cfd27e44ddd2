"""Shared helpers for the GPU parity tests (test infrastructure)."""

from __future__ import annotations

import numpy as np

F32 = np.float32


def rel_err(got: np.ndarray, ref: np.ndarray) -> float:
    """max |got-ref| / max |ref| per trailing vector (per head), worst over all."""
    g = np.asarray(got, np.float64).reshape(-1, got.shape[-1])
    r = np.asarray(ref, np.float64).reshape(-1, ref.shape[-1])
    num = np.abs(g - r).max(axis=1)
    den = np.maximum(np.abs(r).max(axis=1), 1e-30)
    return float((num / den).max())


def elem_rel_err(got, ref, floor: float = 0.0) -> float:
    """max |got-ref| / max(|ref|, floor) elementwise."""
    g = np.asarray(got, np.float64)
    r = np.asarray(ref, np.float64)
    return float((np.abs(g - r) / np.maximum(np.abs(r), max(floor, 1e-30))).max()) if r.size else 0.0


def tol_for(dtype_name: str) -> float:
    """North-star tolerances: 1e-5 relative (fp32), 2e-3 relative (bf16)."""
    return 1e-5 if dtype_name == "f32" else 2e-3
