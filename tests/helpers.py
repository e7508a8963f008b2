"""Shared helpers for the GPU parity tests (inputs from synth/, expectations from oracle/)."""
from __future__ import annotations

import numpy as np
import torch

from synth import round_bf16

TOL = {"f32": 1e-4, "bf16": 2e-2}   # north_star tolerances, metric g17
WEIGHT_KEYS = ("W", "W0", "a", "b", "Wk", "Wq", "Wv", "Watt", "Wmsg", "A")


def rel_err(gpu: np.ndarray, ref: np.ndarray) -> float:
    """|| gpu - ref ||_inf / max(|| ref ||_inf, 1e-30)  (reading g17)."""
    gpu = np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64)
    if ref.size == 0:
        return 0.0
    return float(np.max(np.abs(gpu - ref)) / max(float(np.max(np.abs(ref))), 1e-30))


def prepare(inp: dict, dtype: str) -> dict:
    """Round host inputs to what the device path sees (bf16: round-to-nearest-even, C7)."""
    if dtype == "f32":
        return dict(inp)
    out = {}
    for k, v in inp.items():
        out[k] = round_bf16(v) if (k == "X" or k in WEIGHT_KEYS) else v
    return out


def to_device(inp: dict, dtype: str, device="cuda") -> dict:
    td = torch.float32 if dtype == "f32" else torch.bfloat16
    out = {}
    for k, v in inp.items():
        if k in ("mu", "edge_norm"):
            out[k] = torch.tensor(v, dtype=torch.float32, device=device)
        else:
            out[k] = torch.tensor(np.asarray(v, np.float32), device=device).to(td).contiguous()
    return out
