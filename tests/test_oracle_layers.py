"""Pins of the layer oracle (oracle/layers.py) against things other than itself.

Forward:
  * RGCN identity weights, c = 1, sigma = id on G7: out[q] = h_q+h_a+h_b+h_c+h_p
  * RGCN, one relation, no self-loop, c = 1/sqrt(d_out d_in) == dense GCN A* X W
  * RGCN multi-relation == dense aggregate-then-transform sum_r (C_r o A_r) X W_r
  * RGAT == dense multi-relation GAT in matrix form; HGT == dense masked scaled
    dot-product attention (P:578-588 g-SDDMM + masked row softmax)
  * edge softmax sums to 1 per destination with >= 1 in-edge
  * uniform X and identical relation weights => alpha = 1/in-degree
  * empty rows give zero aggregation
Backward:
  * central finite differences, h = 1e-6, fp64
  * softmax-Jacobian rows sum to zero for any upstream gradient
  * chunked-destination decomposition (oracle/sample.py) reproduces the full gradients
"""
import numpy as np
import pytest

from oracle import layers as L
from oracle import dense as D
from oracle import fd
from oracle import sample as S
from synth import g7, random_small_graph, layer_inputs, upstream_grad, config_graph
from synth.graphs import HeteroGraph


def _rel_err(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


def test_rgcn_identity_g7():
    g = g7()
    X = np.random.default_rng(0).normal(size=(5, 4))
    I = np.eye(4)
    out, _ = L.rgcn_forward(g, X, np.stack([I, I]), I, np.ones(g.num_edges))
    q, a, b, c, p = 4, 0, 1, 2, 3
    assert np.allclose(out[q], X[q] + X[a] + X[b] + X[c] + X[p], atol=1e-14)
    # p receives writes from a, b and cites from q
    assert np.allclose(out[p], X[p] + X[a] + X[b] + X[q], atol=1e-14)
    # authors have no in-edges: self-loop only
    assert np.allclose(out[a], X[a], atol=0)


@pytest.mark.parametrize("seed", range(20))
def test_gcn_reduction(seed):
    g = random_small_graph(seed, max_rels=1)
    g = HeteroGraph(g.node_type_ptr, 1, g.src, g.dst, np.zeros_like(g.rel))
    rng = np.random.default_rng(seed)
    X = rng.normal(size=(g.num_nodes, 5))
    W = rng.normal(size=(1, 5, 3))
    norm = L.rgcn_edge_norm(g, "sym")
    out, _ = L.rgcn_forward(g, X, W, np.zeros((5, 3)), norm, self_loop=False)
    ref = D.gcn_dense(g, X, W[0])
    assert np.allclose(out, ref, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("seed", range(30))
def test_rgcn_dense(seed):
    g = random_small_graph(seed)
    inp = layer_inputs("rgcn", g, 6, 5, seed_x=seed, seed_w=seed + 1)
    norm = L.rgcn_edge_norm(g, "mean")
    out, _ = L.rgcn_forward(g, inp["X"], inp["W"], inp["W0"], norm)
    ref = D.rgcn_dense(g, inp["X"], inp["W"], inp["W0"], norm)
    assert np.allclose(out, ref, rtol=1e-12, atol=1e-12)


def _in_degree(g):
    return np.bincount(g.dst, minlength=g.num_nodes)


@pytest.mark.parametrize("seed", range(30))
def test_rgat_dense(seed):
    g = random_small_graph(seed)
    inp = layer_inputs("rgat", g, 6, 5, seed_x=seed, seed_w=seed + 1)
    out, c = L.rgat_forward(g, inp["X"], inp["W"], inp["a"], inp["b"])
    ref, alpha_cat = D.rgat_dense(g, inp["X"], inp["W"], inp["a"], inp["b"])
    assert np.allclose(out, ref, rtol=1e-12, atol=1e-12)
    assert np.allclose(c["alpha"], D.edge_alpha_from_dense(g, alpha_cat), atol=1e-13)
    # logits as a g-SDDMM: z_e = (X W_r)[src].a_r + (X W_r)[dst].b_r
    for r in range(g.num_rels):
        m = g.rel == r
        if not m.any():
            continue
        sub = HeteroGraph(g.node_type_ptr, g.num_rels, g.src[m], g.dst[m], g.rel[m])
        H = inp["X"] @ inp["W"][r]
        ones = np.ones((g.num_nodes, 1))
        z = D.gsddmm_dense(sub, ones, (H @ inp["a"][r])[:, None]) + D.gsddmm_dense(sub, (H @ inp["b"][r])[:, None], ones)
        assert np.allclose(c["z"][m], z, atol=1e-13)


@pytest.mark.parametrize("seed", range(30))
def test_hgt_dense(seed):
    g = random_small_graph(seed)
    inp = layer_inputs("hgt", g, 6, 4, seed_x=seed, seed_w=seed + 1)
    inp["mu"] = np.random.default_rng(seed).uniform(0.5, 1.5, size=g.num_rels)
    args = [inp[k] for k in ("X", "Wk", "Wq", "Wv", "Watt", "Wmsg", "mu")]
    out, c = L.hgt_forward(g, *args)
    ref, alpha_cat = D.hgt_dense(g, *args)
    assert np.allclose(out, ref, rtol=1e-12, atol=1e-12)
    assert np.allclose(c["alpha"], D.edge_alpha_from_dense(g, alpha_cat), atol=1e-13)


def test_hgt_one_relation_is_masked_attention():
    """R = 1, T = 1, Watt = Wmsg = I: out = softmax_mask(Q K^T / sqrt(d)) V (textbook attention)."""
    g = random_small_graph(7, max_rels=1, max_types=1)
    g = HeteroGraph(np.array([0, g.num_nodes]), 1, g.src, g.dst, np.zeros_like(g.rel))
    rng = np.random.default_rng(3)
    d = 4
    X = rng.normal(size=(g.num_nodes, d))
    Wk, Wq, Wv = (rng.normal(size=(1, d, d)) for _ in range(3))
    I = np.eye(d)[None]
    out, _ = L.hgt_forward(g, X, Wk, Wq, Wv, I, I, np.ones(1))
    Q, K, V = X @ Wq[0], X @ Wk[0], X @ Wv[0]
    A = np.zeros((g.num_nodes, g.num_nodes), bool)
    A[g.dst, g.src] = True
    Lg = np.where(A, Q @ K.T / np.sqrt(d), -np.inf)
    ref = np.zeros_like(out)
    for i in range(g.num_nodes):
        if A[i].any():
            w = np.exp(Lg[i] - Lg[i][A[i]].max())
            w[~A[i]] = 0
            ref[i] = (w / w.sum()) @ V
    assert np.allclose(out, ref, atol=1e-12)


@pytest.mark.parametrize("model", ["rgat", "hgt"])
def test_softmax_sums_to_one_and_uniform(model):
    g = config_graph("tiny", seed=1, scale=0.2)
    inp = layer_inputs(model, g, 8, 8)
    out, c = L.forward(model, g, inp)
    s = np.zeros(g.num_nodes)
    np.add.at(s, g.dst, c["alpha"])
    deg = _in_degree(g)
    assert np.allclose(s[deg > 0], 1.0, atol=1e-12)
    assert np.all(out[deg == 0] == 0.0)           # empty rows: zero aggregation
    # uniform features and identical relation weights -> alpha = 1/in-degree
    u = {k: v.copy() for k, v in inp.items()}
    u["X"][:] = 0.3
    for k in ("W", "a", "b", "Watt", "Wmsg"):
        if k in u:
            u[k][:] = u[k][0]
    for k in ("Wk", "Wq", "Wv"):
        if k in u:
            u[k][:] = u[k][0]
    _, cu = L.forward(model, g, u)
    assert np.allclose(cu["alpha"], 1.0 / deg[g.dst], atol=1e-12)


def test_softmax_backward_rows_sum_to_zero():
    g = config_graph("tiny", seed=2, scale=0.2)
    rng = np.random.default_rng(5)
    l = rng.normal(size=g.num_edges)
    alpha, _, _ = L.edge_softmax(l, g.dst, g.num_nodes)
    dl = L.edge_softmax_backward(alpha, rng.normal(size=g.num_edges), g.dst, g.num_nodes)
    rows = np.zeros(g.num_nodes)
    np.add.at(rows, g.dst, dl)
    assert np.max(np.abs(rows)) < 1e-13


def _fd_check(model, g, d_in, d_out, seed, n_probe=6, opts=None):
    opts = opts or {}
    inp = layer_inputs(model, g, d_in, d_out, seed_x=seed, seed_w=seed + 1)
    G = upstream_grad(g.num_nodes, d_out, seed=seed + 2)
    if model == "rgcn":
        opts.setdefault("norm", L.rgcn_edge_norm(g, "mean"))
    grads = L.backward(model, g, inp, G, **opts)

    def fwd(p):
        return L.forward(model, g, p, **opts)[0]

    rng = np.random.default_rng(seed)
    for name in ("X",) + L.PARAMS[model] + (("A",) if opts.get("tail") else ()):
        if "d" + name not in grads:
            continue
        arr = inp[name]
        idx = [tuple(int(rng.integers(0, s)) for s in arr.shape) for _ in range(n_probe)]
        num = fd.fd_entries(fwd, inp, G, name, idx)
        ana = np.array([grads["d" + name][i] for i in idx])
        err = np.abs(ana - num) / np.maximum(1.0, np.abs(num))
        assert np.max(err) <= 1e-6, (model, name, err)


@pytest.mark.parametrize("model", ["rgcn", "rgat", "hgt"])
def test_fd_g7(model):
    _fd_check(model, g7(), 3, 4, seed=11, n_probe=12)


@pytest.mark.parametrize("model", ["rgcn", "rgat", "hgt"])
@pytest.mark.parametrize("seed", range(8))
def test_fd_random(model, seed):
    g = random_small_graph(100 + seed, allow_multi=(seed % 2 == 1))
    _fd_check(model, g, 5, 4, seed=seed)


def test_fd_rgcn_without_self_loop():
    g = random_small_graph(3)
    _fd_check("rgcn", g, 4, 4, seed=3, opts={"self_loop": False, "norm": L.rgcn_edge_norm(g, "sym")})


@pytest.mark.parametrize("model", ["rgcn", "rgat", "hgt"])
def test_destination_decomposition(model):
    """Sum over destination chunks of (in-edge subgraph, masked G) == full gradients."""
    g = config_graph("tiny", seed=3, scale=0.3)
    inp = layer_inputs(model, g, 8, 8)
    G = upstream_grad(g.num_nodes, 8)
    norm = L.rgcn_edge_norm(g, "mean") if model == "rgcn" else None
    full = L.backward(model, g, inp, G, norm=norm)
    out_full, _ = L.forward(model, g, inp, norm=norm)
    chunks = np.array_split(np.random.default_rng(0).permutation(g.num_nodes), 3)
    acc = {k: np.zeros_like(v) for k, v in full.items()}
    for ch in chunks:
        sub, eids = S.in_edge_subgraph(g, ch)
        kw = {"norm": norm[eids]} if model == "rgcn" else {}
        part = L.backward(model, sub, inp, S.masked_grad(G, ch), **kw)
        for k in acc:
            acc[k] += part[k]
        out_sub, _ = L.forward(model, sub, inp, **kw)
        assert np.allclose(out_sub[ch], out_full[ch], atol=1e-12)
    for k in full:
        assert _rel_err(acc[k], full[k]) < 1e-12, k


# ----------------------------------------------------------------- multi-head HGT (F2, reading b12)
@pytest.mark.parametrize("heads", [2, 4])
@pytest.mark.parametrize("seed", range(4))
def test_hgt_head_logits_and_softmax(heads, seed):
    """Per head h: the logit is mu_r K'[:, h] . q[:, h] / sqrt(dh), its softmax sums to one per
    destination, and out[:, h] is the alpha_h-weighted sum of M[:, h] (brute force per edge)."""
    g = random_small_graph(300 + seed, allow_multi=True)
    d = 8
    inp = layer_inputs("hgt", g, 5, d, seed_x=seed, seed_w=seed + 1)
    mu = inp["mu"] * 1.3
    out, c = L.hgt_forward(g, inp["X"], inp["Wk"], inp["Wq"], inp["Wv"], inp["Watt"], inp["Wmsg"], mu, heads=heads)
    dh = d // heads
    Kp, q, M = c["Kp"], c["q"], c["M"]
    for h in range(heads):
        cs = slice(h * dh, (h + 1) * dh)
        want = mu[g.rel] * np.sum(Kp[:, cs] * q[:, cs], axis=1) / np.sqrt(dh)
        np.testing.assert_allclose(c["logit"][:, h], want, rtol=1e-12, atol=1e-12)
        for v in range(g.num_nodes):
            es = np.nonzero(g.dst == v)[0]
            if len(es) == 0:
                assert np.all(out[v, cs] == 0)
                continue
            ex = np.exp(want[es] - want[es].max())
            a = ex / ex.sum()
            np.testing.assert_allclose(out[v, cs], (a[:, None] * M[es][:, cs]).sum(0), rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("heads", [2, 4])
def test_hgt_heads_one_relation_reduce_to_single_head(heads):
    from synth.graphs import HeteroGraph
    rng = np.random.default_rng(7)
    n, E = 12, 40
    g = HeteroGraph(np.array([0, 5, n]), 1, rng.integers(0, n, E).astype(np.int32),
                    rng.integers(0, n, E).astype(np.int32), np.zeros(E, np.int32))
    d = 8
    inp = layer_inputs("hgt", g, 6, d, seed_x=1, seed_w=2)
    out, _ = L.hgt_forward(g, inp["X"], inp["Wk"], inp["Wq"], inp["Wv"], inp["Watt"], inp["Wmsg"], inp["mu"],
                           heads=heads)
    dh = d // heads
    I = np.eye(dh)[None]
    for h in range(heads):
        cs = slice(h * dh, (h + 1) * dh)
        Wk1 = inp["Wk"] @ inp["Watt"][0][:, cs]
        Wv1 = inp["Wv"] @ inp["Wmsg"][0][:, cs]
        o1, _ = L.hgt_forward(g, inp["X"], Wk1, inp["Wq"][:, :, cs], Wv1, I, I, inp["mu"])
        np.testing.assert_allclose(out[:, cs], o1, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("heads", [2, 4])
@pytest.mark.parametrize("seed", range(3))
def test_fd_hgt_heads(heads, seed):
    g = random_small_graph(400 + seed, allow_multi=True)
    _fd_check("hgt", g, 5, 8, seed=seed, opts={"heads": heads})


# ----------------------------------------------------------------- HGT tail (F2, reading b12)
def test_gelu_values():
    """GELU(x) = x Phi(x): Phi(1) = 0.8413447460685429, Phi(-1) = 0.15865525393145707 (normal CDF
    table values), GELU(0) = 0, GELU(x) -> x for large x and -> 0 for very negative x."""
    x = np.array([0.0, 1.0, -1.0, 2.0, 8.0, -8.0])
    want = np.array([0.0, 0.8413447460685429, -0.15865525393145707, 2 * 0.9772498680518208, 8.0, 0.0])
    np.testing.assert_allclose(L.gelu(x), want, rtol=1e-12, atol=1e-12)
    # derivative: Phi(x) + x phi(x); at 0 it is 1/2, at 1: 0.8413447 + 0.2419707
    np.testing.assert_allclose(L.gelu_grad(np.array([0.0, 1.0])), [0.5, 0.8413447460685429 + 0.24197072451914337],
                               rtol=1e-12)


def test_tail_identity_weights():
    g = random_small_graph(31)
    rng = np.random.default_rng(1)
    h = rng.normal(size=(g.num_nodes, 4))
    I = np.broadcast_to(np.eye(4), (g.num_node_types, 4, 4))
    np.testing.assert_allclose(L.hgt_tail_forward(g, h, np.zeros_like(h), I), L.gelu(h), rtol=1e-13)
    X = rng.normal(size=h.shape)
    np.testing.assert_allclose(L.hgt_tail_forward(g, h, X, I) - X, L.gelu(h), rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("heads", [1, 2])
@pytest.mark.parametrize("seed", range(3))
def test_fd_hgt_tail(heads, seed):
    g = random_small_graph(500 + seed, allow_multi=True)
    _fd_check("hgt", g, 8, 8, seed=seed, opts={"heads": heads, "tail": True})


# ----------------------------------------------------------------- RGCN normaliser c_{v,r} (reading g1)
def _golden(name):
    import json
    import os
    return json.load(open(os.path.join(os.path.dirname(__file__), "golden", name)))


def _frac(s):
    from fractions import Fraction
    import math
    if s.startswith("1/sqrt("):
        return 1.0 / math.sqrt(int(s[len("1/sqrt("):-1]))
    return float(Fraction(s))


@pytest.mark.parametrize("kind", ["mean", "sym"])
def test_rgcn_norm_g7_hand_values(kind):
    """Eq. 3.1's 1/c_{v,r} on G7, values worked by hand (tests/golden/g7_rgcn_norm.json)."""
    gold = _golden("g7_rgcn_norm.json")
    want = np.array([_frac(s) for s in gold[f"{kind}_by_eid"]])
    got = L.rgcn_edge_norm(g7(), kind)
    assert np.allclose(got, want, rtol=0, atol=1e-15)


def test_rgcn_mean_identity_ones_g7():
    """mean norm, X = 1, W_r = I, W_0 = 0: out_v = #relations with an in-edge into v (hand value)."""
    g = g7()
    gold = _golden("g7_rgcn_norm.json")["rgcn_mean_identity_ones"]["out"]
    I = np.eye(3)
    out, _ = L.rgcn_forward(g, np.ones((5, 3)), np.stack([I, I]), np.zeros((3, 3)), L.rgcn_edge_norm(g, "mean"))
    assert np.allclose(out, np.array(gold, float)[:, None] * np.ones((1, 3)), atol=1e-15)


@pytest.mark.parametrize("seed", range(20))
def test_rgcn_mean_is_row_normalised_relation_adjacency(seed):
    """'mean' == sum_r D_r^-1 A_r X W_r + X W_0 with A_r the dense per-relation adjacency (edge
    multiplicities counted) and D_r its row sums, built here from the edge list, not from
    rgcn_edge_norm; a norm over the total in-degree (a plausible slip) fails this."""
    g = random_small_graph(seed, allow_multi=seed % 2 == 1)
    rng = np.random.default_rng(100 + seed)
    n, R = g.num_nodes, g.num_rels
    X = rng.normal(size=(n, 4))
    W = rng.normal(size=(R, 4, 3))
    W0 = rng.normal(size=(4, 3))
    ref = X @ W0
    for r in range(R):
        A = np.zeros((n, n))
        for s_, d_, r_ in zip(g.src, g.dst, g.rel):
            if r_ == r:
                A[d_, s_] += 1.0
        rows = A.sum(axis=1)
        Dinv = np.divide(1.0, rows, out=np.zeros(n), where=rows > 0)
        ref = ref + (Dinv[:, None] * A) @ X @ W[r]
    out, _ = L.rgcn_forward(g, X, W, W0, L.rgcn_edge_norm(g, "mean"))
    assert np.allclose(out, ref, rtol=1e-12, atol=1e-12)
    # and the per-(v, r) weights sum to one
    norm = L.rgcn_edge_norm(g, "mean")
    tot = {}
    for e in range(g.num_edges):
        k = (int(g.dst[e]), int(g.rel[e]))
        tot[k] = tot.get(k, 0.0) + norm[e]
    assert all(abs(v - 1.0) < 1e-12 for v in tot.values())
