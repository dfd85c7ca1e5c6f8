"""Shared test helpers: the parity metric and thin device wrappers (no method arithmetic)."""
from __future__ import annotations

import numpy as np


def rel_err(gpu: np.ndarray, ref: np.ndarray) -> float:
    """Parity metric (R15): max over (g, slot, comp) of |gpu - ref| / R_g^c,
    R_g^c = sum over slots of |ref[g, :, c]| (global row-abs-sum).  Rows with R = 0 must be
    exactly zero on the GPU (returns inf otherwise)."""
    gpu = gpu.reshape(ref.shape)
    R = np.abs(ref).sum(axis=1, keepdims=True)
    diff = np.abs(gpu - ref)
    zero = (R == 0)
    if np.any(zero & (diff > 0)):
        return float("inf")
    with np.errstate(invalid="ignore", divide="ignore"):
        e = np.where(zero, 0.0, diff / np.where(zero, 1.0, R))
    return float(e.max()) if e.size else 0.0


def to_dev(d: dict, device="cuda"):
    import torch
    return {k: torch.from_numpy(np.ascontiguousarray(v)).to(device) for k, v in d.items()}
