"""Seeded layer inputs (features, weights, upstream gradient).

Distributions: X ~ U(-1,1); typed weight matrices
Glorot-uniform +-sqrt(6/(fan_in+fan_out)); RGAT attention vectors ~ U(-1,1)/sqrt(d);
HGT relation prior mu_r = 1 (reading g7, not trained); upstream gradient
G = dL/dout ~ U(-1,1) (reading g12: loss L = sum(out * G)).

Seeds: graph 1, X 2, W 3, G 4 (D1).  Everything is float64 on the host; the
bf16 path receives `round_bf16` copies (round-to-nearest-even), and the oracle
evaluates the same rounded values.
"""
from __future__ import annotations

from typing import Dict

import numpy as np

from .graphs import HeteroGraph


def _glorot(rng, shape, fan_in, fan_out):
    lim = np.sqrt(6.0 / (fan_in + fan_out))
    return rng.uniform(-lim, lim, size=shape)


def layer_inputs(model: str, g: HeteroGraph, d_in: int, d_out: int,
                 seed_x: int = 2, seed_w: int = 3) -> Dict[str, np.ndarray]:
    """Features and weights for one layer of `model` in {'rgcn','rgat','hgt'}."""
    n, r, t = g.num_nodes, g.num_rels, g.num_node_types
    rx = np.random.default_rng(seed_x)
    rw = np.random.default_rng(seed_w)
    out: Dict[str, np.ndarray] = {"X": rx.uniform(-1.0, 1.0, size=(n, d_in))}
    if model == "rgcn":
        out["W"] = _glorot(rw, (r, d_in, d_out), d_in, d_out)
        out["W0"] = _glorot(rw, (d_in, d_out), d_in, d_out)
    elif model == "rgat":
        out["W"] = _glorot(rw, (r, d_in, d_out), d_in, d_out)
        out["a"] = rw.uniform(-1.0, 1.0, size=(r, d_out)) / np.sqrt(d_out)
        out["b"] = rw.uniform(-1.0, 1.0, size=(r, d_out)) / np.sqrt(d_out)
    elif model == "hgt":
        out["Wk"] = _glorot(rw, (t, d_in, d_out), d_in, d_out)
        out["Wq"] = _glorot(rw, (t, d_in, d_out), d_in, d_out)
        out["Wv"] = _glorot(rw, (t, d_in, d_out), d_in, d_out)
        out["Watt"] = _glorot(rw, (r, d_out, d_out), d_out, d_out)
        out["Wmsg"] = _glorot(rw, (r, d_out, d_out), d_out, d_out)
        out["mu"] = np.ones(r)
        out["A"] = _glorot(rw, (t, d_out, d_out), d_out, d_out)  # tail A-linear (F2), drawn last
    else:
        raise ValueError(f"unknown model {model!r}")
    return out


def upstream_grad(n: int, d_out: int, seed: int = 4) -> np.ndarray:
    return np.random.default_rng(seed).uniform(-1.0, 1.0, size=(n, d_out))


def round_bf16(x: np.ndarray) -> np.ndarray:
    """Round float64 values to the nearest bf16 value (ties to even), returned as float64.
    Goes through float32 first (exact for these magnitudes), then rounds the
    float32 bit pattern to its upper 16 bits."""
    f = np.ascontiguousarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    u = (u + 0x7FFF + lsb) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """uint16 bf16 bit patterns of round_bf16(x) (for uploading to the device)."""
    f = round_bf16(x).astype(np.float32)
    return (f.view(np.uint32) >> 16).astype(np.uint16)


def segment_inputs(seed: int, seg_lens, K: int, N: int, num_src: int = 0, num_weights: int = 0,
                   gather: bool = True, shuffle_weights: bool = False) -> Dict[str, np.ndarray]:
    """Inputs of one A1 typed segment GEMM (Y[S] = X[G] x W[T]): segment row offsets from
    `seg_lens` (zeros allowed = empty segments), X ~ U(-1,1) [num_src, K], Glorot W [nw, K, N],
    a uniform random gather index per row (or none), and optionally a random weight per segment."""
    rng = np.random.default_rng(seed)
    seg_ptr = np.concatenate([[0], np.cumsum(np.asarray(seg_lens, np.int64))]).astype(np.int64)
    rows = int(seg_ptr[-1])
    S = len(seg_lens)
    nw = num_weights or S
    num_src = num_src or max(rows, 1)
    out: Dict[str, np.ndarray] = {
        "seg_ptr": seg_ptr,
        "X": rng.uniform(-1.0, 1.0, size=(num_src, K)),
        "W": _glorot(rng, (nw, K, N), K, N),
        "gather": rng.integers(0, num_src, size=rows).astype(np.int32) if gather else None,
        "seg_weight": rng.integers(0, nw, size=S).astype(np.int32) if shuffle_weights else None,
    }
    return out


def random_labels(n: int, num_classes: int, seed: int = 5, labelled_frac: float = 1.0) -> np.ndarray:
    """The "precomputed random label tensor" of the training measurement: int32 class
    ids uniform in [0, num_classes); a seeded (1 - labelled_frac) share of rows gets -1 (no label)."""
    rng = np.random.default_rng(seed)
    y = rng.integers(0, num_classes, size=n).astype(np.int32)
    if labelled_frac < 1.0:
        y[rng.random(n) >= labelled_frac] = -1
    return y


def stack_inputs(model: str, g: HeteroGraph, d: int, num_layers: int) -> list:
    """Weights of `num_layers` stacked layers of width d (layer i drawn with seed 3 + i, D1);
    X (seed 2) is returned in the first layer's dict."""
    out = []
    for i in range(num_layers):
        p = layer_inputs(model, g, d, d, seed_w=3 + i)
        if i:
            p.pop("X")
        out.append(p)
    return out

