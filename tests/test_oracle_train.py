"""Pins of the F4 training-step oracle (oracle/train.py) against things other than itself.

  * NLL loss == a pure-Python loop of -log(exp(z_y) / sum_j exp(z_j)) with math.exp / math.log
    (brute force on tiny inputs), mean over labelled rows
  * uniform logits => L = log C exactly (closed form); rows of dL/dz sum to 0; unlabelled rows
    have zero gradient; no labelled row => L = 0
  * dL/dz and the stacked-layer weight gradients == central finite differences of the loss
    (h = 1e-6, fp64), for RGCN / RGAT / HGT, 1 and 2 layers, with ReLU between
  * a 1-layer stack's gradient == the layer oracle's backward with G = dL/dout (the chain rule
    through an independently written loss)
  * SGD: L(theta - lr g) - L(theta) = -lr |g|^2 + O(lr^2) (first-order decrease; reading b15)
"""
import math

import numpy as np
import pytest

from oracle import layers as L
from oracle import train as T
from synth import g7, random_labels, random_small_graph, stack_inputs

TRAINED = {"rgcn": ("W", "W0"), "rgat": ("W", "a", "b"), "hgt": ("Wk", "Wq", "Wv", "Watt", "Wmsg")}


def _brute_nll(z, y):
    tot, cnt = 0.0, 0
    for i in range(z.shape[0]):
        if not (0 <= y[i] < z.shape[1]):
            continue
        s = sum(math.exp(float(v)) for v in z[i])
        tot += -math.log(math.exp(float(z[i][y[i]])) / s)
        cnt += 1
    return tot / cnt if cnt else 0.0


@pytest.mark.parametrize("seed", range(10))
def test_nll_brute_force(seed):
    rng = np.random.default_rng(seed)
    n, c = int(rng.integers(1, 12)), int(rng.integers(2, 9))
    z = rng.normal(scale=3.0, size=(n, c))
    y = rng.integers(-1, c, size=n)
    loss, grad = T.nll_loss(z, y)
    assert abs(loss - _brute_nll(z, y)) <= 1e-12 * max(1.0, abs(loss))
    # gradient against central differences of the brute-force loss
    h = 1e-6
    for i in range(n):
        for j in range(c):
            zp, zm = z.copy(), z.copy()
            zp[i, j] += h
            zm[i, j] -= h
            fd = (_brute_nll(zp, y) - _brute_nll(zm, y)) / (2 * h)
            assert abs(grad[i, j] - fd) <= 1e-7


def test_nll_closed_forms():
    c = 7
    z = np.full((5, c), 0.37)
    y = np.array([0, 3, 6, 2, 1])
    loss, grad = T.nll_loss(z, y)
    assert abs(loss - math.log(c)) <= 1e-15
    assert np.allclose(grad.sum(axis=1), 0.0, atol=1e-16)
    assert np.allclose(grad[np.arange(5), y], (1.0 / c - 1.0) / 5, atol=1e-16)
    # unlabelled rows: no loss term, no gradient
    y2 = np.array([0, -1, 6, -1, 1])
    loss2, grad2 = T.nll_loss(z, y2)
    assert abs(loss2 - math.log(c)) <= 1e-15
    assert np.all(grad2[[1, 3]] == 0.0)
    assert np.allclose(grad2[[0, 2, 4]].sum(), 0.0, atol=1e-15)
    loss3, grad3 = T.nll_loss(z, np.full(5, -1))
    assert loss3 == 0.0 and not grad3.any()
    # large logits: the max shift keeps it finite and exact
    zz = np.array([[1000.0, 0.0], [0.0, -1000.0]])
    l4, _ = T.nll_loss(zz, np.array([1, 0]))
    assert abs(l4 - 0.5 * (1000.0 + 0.0)) <= 1e-9


def _stack(model, g, d, layers):
    ps = stack_inputs(model, g, d, layers)
    X = ps[0].pop("X")
    return X, ps


@pytest.mark.parametrize("model", ["rgcn", "rgat", "hgt"])
@pytest.mark.parametrize("layers", [1, 2])
@pytest.mark.parametrize("seed", [0, 1])
def test_stack_gradients_fd(model, layers, seed):
    g = random_small_graph(seed + 3, max_nodes=12, max_edges=40)
    d = 4
    X, ps = _stack(model, g, d, layers)
    y = random_labels(g.num_nodes, d, seed=seed, labelled_frac=0.7)
    loss, grads = T.stack_backward(model, g, X, ps, y)
    h = 1e-6
    rng = np.random.default_rng(seed)
    for li in range(layers):
        for k in TRAINED[model]:
            for _ in range(4):
                idx = tuple(int(rng.integers(0, s)) for s in ps[li][k].shape)
                pp = [dict(p) for p in ps]
                pp[li] = {kk: v.copy() for kk, v in ps[li].items()}
                pp[li][k][idx] += h
                lp, _ = T.stack_forward(model, g, X, pp, y)
                pp[li][k][idx] -= 2 * h
                lm, _ = T.stack_forward(model, g, X, pp, y)
                fd = (lp - lm) / (2 * h)
                an = grads[li]["d" + k][idx]
                assert abs(an - fd) <= 1e-6 * max(1.0, abs(fd)), (li, k, idx, an, fd)


def test_one_layer_chain_rule():
    g = g7()
    X, ps = _stack("hgt", g, 4, 1)
    y = np.array([0, 1, 2, 3, -1], np.int32)
    loss, grads = T.stack_backward("hgt", g, X, ps, y)
    out, _ = L.forward("hgt", g, dict(ps[0], X=X))
    _, G = T.nll_loss(out, y)
    ref = L.backward("hgt", g, dict(ps[0], X=X), G)
    for k in TRAINED["hgt"]:
        assert np.allclose(grads[0]["d" + k], ref["d" + k], rtol=0, atol=0)


@pytest.mark.parametrize("model", ["rgcn", "rgat", "hgt"])
def test_sgd_first_order_decrease(model):
    g = random_small_graph(11, max_nodes=16, max_edges=60)
    X, ps = _stack(model, g, 8, 2)
    y = random_labels(g.num_nodes, 8, seed=2)
    lr = 1e-4
    loss, grads, new = T.train_step(model, g, X, ps, y, lr, TRAINED[model])
    l1, _ = T.stack_forward(model, g, X, new, y)
    gn2 = sum(float(np.sum(gr["d" + k] ** 2)) for gr in grads for k in TRAINED[model])
    assert gn2 > 0
    assert l1 < loss
    assert abs((l1 - loss) - (-lr * gn2)) <= 1e-2 * lr * gn2
    # untrained entries (HGT mu) are untouched; trained ones moved by exactly lr * grad
    for p, q, gr in zip(ps, new, grads):
        for k in p:
            if k in TRAINED[model]:
                assert np.array_equal(q[k], p[k] - lr * gr["d" + k])
            else:
                assert q[k] is p[k]


def test_act_round_identity_and_effect():
    """act_round = identity reproduces the unrounded stack; bf16 rounding changes the loss by
    O(2^-9) only (it rounds the second layer's input, C7)."""
    from synth import round_bf16
    g = random_small_graph(5, max_nodes=16, max_edges=60)
    X, ps = _stack("rgat", g, 8, 2)
    y = random_labels(g.num_nodes, 8, seed=1)
    l0, g0 = T.stack_backward("rgat", g, X, ps, y)
    l1, g1 = T.stack_backward("rgat", g, X, ps, y, act_round=lambda a: a)
    assert l0 == l1 and all(np.array_equal(a["dW"], b["dW"]) for a, b in zip(g0, g1))
    l2, _ = T.stack_backward("rgat", g, X, ps, y, act_round=round_bf16)
    assert l2 != l0 and abs(l2 - l0) <= 1e-2 * abs(l0)
