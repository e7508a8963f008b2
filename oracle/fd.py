"""Central finite differences of L = sum(out * G) (reading g12), float64.

TEST INFRASTRUCTURE (see oracle/__init__.py).  Pins the analytic backward of
oracle/layers.py (central differences, h = 1e-6, relative
error <= 1e-4).  Works for any forward callable; independent of the backward code.
"""
from __future__ import annotations

from typing import Callable, Dict, Iterable, Tuple

import numpy as np


def loss(out: np.ndarray, G: np.ndarray) -> float:
    return float(np.sum(out * G))


def fd_entries(fwd: Callable[[Dict[str, np.ndarray]], np.ndarray], params: Dict[str, np.ndarray],
               G: np.ndarray, name: str, indices: Iterable[Tuple[int, ...]], h: float = 1e-6) -> np.ndarray:
    """dL/dparams[name][idx] for each idx by central differences."""
    if h <= 0:
        raise ValueError("h must be positive")
    vals = []
    for idx in indices:
        p = {k: v.copy() for k, v in params.items()}
        p[name][idx] += h
        lp = loss(fwd(p), G)
        p[name][idx] -= 2 * h
        lm = loss(fwd(p), G)
        if not (np.isfinite(lp) and np.isfinite(lm)):
            raise FloatingPointError("non-finite loss")
        vals.append((lp - lm) / (2 * h))
    return np.asarray(vals)
