"""fp64 oracle of the F4 training step: stacked RGNN layers, NLL loss, SGD update.

TEST INFRASTRUCTURE (see oracle/__init__.py).  SURVEY.md §8(f) F4: "end-to-end
2-layer training step (NLL loss vs random labels, SGD update)".  The paper's
training measurement: "to obtain a loss, we compute the negative log-likelihood
loss by comparing the output with a precomputed random label tensor" (P:1062
§3.4.1); the BASELINE.json AIFB/AM configs are "RGAT 2 layers hidden 64".

Readings (DESIGN.md b13-b15):
  * between stacked layers: ReLU, h_{l+1} input = max(h_l, 0); on the bf16
    path the next layer reads the bf16 rounding of max(h_l, 0), so the oracle of that path
    applies the same rounding (`act_round`), as C7 rounds the first layer's X;
  * loss: L = -(1/|V_lab|) sum_{v in V_lab} log softmax(out_v)[y_v] over the rows with a
    label y_v in [0, C) (rows with y_v < 0 carry no label), the negative log-likelihood of
    log_softmax outputs, mean reduction;
  * optimiser: plain SGD, theta <- theta - lr * dL/dtheta (no momentum, no weight decay),
    applied to every trained weight of every layer (HGT mu is not trained, g7).

Everything is evaluated by the layer oracle (oracle/layers.py) and plain numpy,
in float64, with no fusion: layer 1, ReLU, layer 2, log-softmax, NLL, then the
exact backward in reverse order, then the update.
"""
from __future__ import annotations

from typing import Callable, Dict, List, Optional, Sequence, Tuple

import numpy as np

from synth.graphs import HeteroGraph

from . import layers as L


def relu(x: np.ndarray) -> np.ndarray:
    return np.maximum(x, 0.0)


def log_softmax(z: np.ndarray) -> np.ndarray:
    """log softmax over the last axis, max-shifted (mathematically the plain definition)."""
    m = z.max(axis=-1, keepdims=True)
    return z - m - np.log(np.exp(z - m).sum(axis=-1, keepdims=True))


def nll_loss(logits: np.ndarray, labels: np.ndarray) -> Tuple[float, np.ndarray]:
    """Mean negative log-likelihood of log_softmax(logits) at the labels, over
    the rows with a label in [0, C); returns (L, dL/dlogits).
    dL/dz_v = (softmax(z_v) - onehot(y_v)) / |V_lab| for labelled rows, 0 otherwise."""
    n, c = logits.shape
    lab = np.asarray(labels)
    rows = np.nonzero((lab >= 0) & (lab < c))[0]
    grad = np.zeros_like(logits, dtype=np.float64)
    if rows.size == 0:
        return 0.0, grad
    lp = log_softmax(logits[rows])
    loss = -float(lp[np.arange(rows.size), lab[rows]].sum()) / rows.size
    p = np.exp(lp)
    p[np.arange(rows.size), lab[rows]] -= 1.0
    grad[rows] = p / rows.size
    return loss, grad


def _layer_inp(params: Dict[str, np.ndarray], X: np.ndarray) -> Dict[str, np.ndarray]:
    d = dict(params)
    d["X"] = X
    return d


Round = Optional[Callable[[np.ndarray], np.ndarray]]


def _act(h: np.ndarray, act_round: Round) -> np.ndarray:
    a = relu(h)
    return act_round(a) if act_round is not None else a


def stack_forward(model: str, g: HeteroGraph, X: np.ndarray, params: Sequence[Dict[str, np.ndarray]],
                  labels: np.ndarray, act_round: Round = None, **kw) -> Tuple[float, List[np.ndarray]]:
    """Forward of len(params) stacked layers with ReLU between them, then the NLL loss.
    Returns (loss, [h_1, ..., h_n]) (pre-activation layer outputs)."""
    hs: List[np.ndarray] = []
    x = X
    for i, p in enumerate(params):
        h, _ = L.forward(model, g, _layer_inp(p, x), **kw)
        hs.append(h)
        x = _act(h, act_round) if i + 1 < len(params) else h
    loss, _ = nll_loss(hs[-1], labels)
    return loss, hs


def stack_backward(model: str, g: HeteroGraph, X: np.ndarray, params: Sequence[Dict[str, np.ndarray]],
                   labels: np.ndarray, act_round: Round = None, **kw) -> Tuple[float, List[Dict[str, np.ndarray]]]:
    """Loss and the weight gradients of every layer (list of dicts in layer order).
    Layer 1's dX (the input features) is dropped: the input is data, not a parameter.
    With act_round the rounding is treated as the identity in the backward (straight through:
    the gradient flows to max(h, 0) unchanged, as on the device)."""
    loss, hs = stack_forward(model, g, X, params, labels, act_round, **kw)
    _, G = nll_loss(hs[-1], labels)
    grads: List[Dict[str, np.ndarray]] = [None] * len(params)  # type: ignore[list-item]
    for i in range(len(params) - 1, -1, -1):
        x = X if i == 0 else _act(hs[i - 1], act_round)
        gi = L.backward(model, g, _layer_inp(params[i], x), G, **kw)
        if i > 0:
            G = gi["dX"] * (hs[i - 1] > 0)   # ReLU' (0 at h = 0)
        gi.pop("dX", None)
        grads[i] = gi
    return loss, grads


def sgd(params: Sequence[Dict[str, np.ndarray]], grads: Sequence[Dict[str, np.ndarray]], lr: float,
        trained: Sequence[str]) -> List[Dict[str, np.ndarray]]:
    """theta <- theta - lr * grad for every trained weight (reading b15)."""
    out = []
    for p, g in zip(params, grads):
        q = dict(p)
        for k in trained:
            q[k] = p[k] - lr * g["d" + k]
        out.append(q)
    return out


def train_step(model: str, g: HeteroGraph, X: np.ndarray, params: Sequence[Dict[str, np.ndarray]],
               labels: np.ndarray, lr: float, trained: Sequence[str], act_round: Round = None, **kw):
    """One training step: returns (loss before the update, grads, updated params)."""
    loss, grads = stack_backward(model, g, X, params, labels, act_round, **kw)
    return loss, grads, sgd(params, grads, lr, trained)
