"""A1 typed segment GEMM, Y[S] = X[G] x W[T] (the paper's GEMM template, §3.3.3;
algo:gemm_template P:901-918), in float64.

TEST INFRASTRUCTURE (see oracle/__init__.py).  Rows 0..R-1 are split into contiguous
segments by seg_ptr; every row i of segment s is  Y[i] = X[G(i)] . W[w(s)]  with
G(i) = gather[i] (identity when gather is None) and w(s) = seg_weight[s] (s when None)
-- the template's "gather list" G and "type" T (X[G] gathers rows, W[T] picks the
weight of the row's segment).  One numpy matmul per segment is the only library step.
"""
from __future__ import annotations

from typing import Optional

import numpy as np


def segment_gemm(X: np.ndarray, W: np.ndarray, seg_ptr: np.ndarray, gather: Optional[np.ndarray] = None,
                 seg_weight: Optional[np.ndarray] = None, trans_w: bool = False) -> np.ndarray:
    """Y[seg_ptr[-1], N]: for each segment s, Y[rows of s] = X[G(rows of s)] @ W[w(s)]
    (W[w(s)].T when trans_w, i.e. W stored as [num_weights][N][K])."""
    X = np.asarray(X, np.float64)
    W = np.asarray(W, np.float64)
    seg_ptr = np.asarray(seg_ptr, np.int64)
    N = W.shape[1] if trans_w else W.shape[2]
    rows = int(seg_ptr[-1])
    Y = np.zeros((rows, N))
    for s in range(len(seg_ptr) - 1):
        lo, hi = int(seg_ptr[s]), int(seg_ptr[s + 1])
        if hi == lo:
            continue
        idx = np.arange(lo, hi) if gather is None else np.asarray(gather[lo:hi], np.int64)
        w = s if seg_weight is None else int(seg_weight[s])
        Ws = W[w].T if trans_w else W[w]
        Y[lo:hi] = X[idx] @ Ws
    return Y
