"""Pins of oracle/gemm.py (A1 typed segment GEMM) against things other than itself:
brute-force triple loops on tiny inputs, the per-edge messages of the GEMM template's
vanilla materialization, and the single-segment special case."""
import numpy as np
import pytest

from oracle import gemm as og
from oracle import graph as ograph
from synth import random_small_graph, segment_inputs


def _brute(X, W, seg_ptr, gather, seg_weight, trans_w):
    rows = int(seg_ptr[-1])
    N = W.shape[1] if trans_w else W.shape[2]
    K = X.shape[1]
    Y = [[0.0] * N for _ in range(rows)]
    s = 0
    for i in range(rows):
        while not (seg_ptr[s] <= i < seg_ptr[s + 1]):
            s += 1
        src = i if gather is None else int(gather[i])
        w = s if seg_weight is None else int(seg_weight[s])
        for n in range(N):
            acc = 0.0
            for k in range(K):
                acc += X[src][k] * (W[w][n][k] if trans_w else W[w][k][n])
            Y[i][n] = acc
    return np.array(Y).reshape(rows, N)


@pytest.mark.parametrize("seed", range(12))
def test_brute_force(seed):
    rng = np.random.default_rng(100 + seed)
    lens = rng.integers(0, 5, size=rng.integers(1, 6))
    K, N = int(rng.integers(1, 6)), int(rng.integers(1, 5))
    inp = segment_inputs(seed, lens, K, N, num_src=max(7, int(np.sum(lens))), num_weights=len(lens) + 1, gather=bool(seed % 2),
                         shuffle_weights=seed % 3 == 0)
    trans = seed % 4 == 1
    W = np.ascontiguousarray(np.swapaxes(inp["W"], 1, 2)) if trans else inp["W"]
    X = inp["X"] if inp["gather"] is not None else inp["X"][: int(inp["seg_ptr"][-1])]
    if X.shape[0] == 0:
        X = np.zeros((1, K))
    got = og.segment_gemm(X, W, inp["seg_ptr"], inp["gather"], inp["seg_weight"], trans_w=trans)
    want = _brute(X, W, inp["seg_ptr"], inp["gather"], inp["seg_weight"], trans)
    assert got.shape == want.shape
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-12)


def test_single_segment_is_plain_matmul():
    rng = np.random.default_rng(5)
    X, W = rng.standard_normal((9, 4)), rng.standard_normal((1, 4, 3))
    np.testing.assert_allclose(og.segment_gemm(X, W, np.array([0, 9])), X @ W[0], rtol=1e-13)


@pytest.mark.parametrize("seed", range(5))
def test_compact_rows_reproduce_per_edge_messages(seed):
    """Over the compact pairs (C1 build, segments = relations, G = pair_src) the GEMM rows are
    the per-edge messages X[s_e] W_{r_e} of vanilla materialization: row
    edge_pair[e] equals the message of edge e, computed edge by edge."""
    g = random_small_graph(40 + seed, allow_multi=True)
    b = ograph.build(g.num_nodes, g.num_rels, g.src, g.dst, g.rel)
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((g.num_nodes, 5))
    W = rng.standard_normal((g.num_rels, 5, 3))
    Y = og.segment_gemm(X, W, np.asarray(b["pair_rel_ptr"]), np.asarray(b["pair_src"]))
    for e in range(g.num_edges):
        msg = np.array([sum(X[g.src[e], k] * W[g.rel[e], k, n] for k in range(5)) for n in range(3)])
        np.testing.assert_allclose(Y[b["edge_pair"][e]], msg, rtol=1e-12, atol=1e-12)
