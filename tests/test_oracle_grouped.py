"""Cross-check of the two oracle modes: the C/OpenMP "grouped" oracle
(oracle/grouped.c: one product per distinct (relation, node) pair, exact by P:775 §3.3.2) against
the per-edge numpy oracle (oracle/layers.py, itself pinned by tests/test_oracle_layers.py) on tiny,
AIFB- and BGS-shaped graphs, every output and gradient, at fp64 rounding level.  The grouped mode is
what bench.py times on full-size graphs, so this is what makes that timing a timing of the oracle."""
import numpy as np
import pytest

from oracle import grouped as OG
from oracle import layers as L
from synth import config_graph, layer_inputs, upstream_grad, g7


def _rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


CASES = [("tiny", 0.3), ("aifb", 0.5), ("bgs", 0.05)]


@pytest.mark.parametrize("model", ["rgcn", "rgat", "hgt"])
@pytest.mark.parametrize("graph,scale", CASES)
@pytest.mark.parametrize("threads", [1, 4])
def test_grouped_matches_per_edge(model, graph, scale, threads):
    g = config_graph(graph, seed=1, scale=scale)
    d = 16
    inp = layer_inputs(model, g, d, d)
    G = upstream_grad(g.num_nodes, d)
    kw = {}
    if model == "rgcn":
        kw["norm"] = L.rgcn_edge_norm(g, "mean")
    ref_out, _ = L.forward(model, g, inp, **kw)
    ref = L.backward(model, g, inp, G, **kw)
    OG.set_threads(threads)
    out, grads = OG.forward_backward(model, g, inp, G, **kw)
    assert _rel(out, ref_out) < 1e-12
    assert set(grads) == set(ref), (set(grads), set(ref))
    for k in ref:
        assert _rel(grads[k], ref[k]) < 1e-11, (k, _rel(grads[k], ref[k]))


def test_grouped_g7_multi_edge_and_empty_rows():
    """G7 has empty rows and shared pairs; add a duplicate edge (g11: each contributes)."""
    g = g7()
    g.src = np.concatenate([g.src, g.src[:1]]).astype(np.int32)
    g.dst = np.concatenate([g.dst, g.dst[:1]]).astype(np.int32)
    g.rel = np.concatenate([g.rel, g.rel[:1]]).astype(np.int32)
    for model in ("rgcn", "rgat", "hgt"):
        inp = layer_inputs(model, g, 3, 3)
        G = upstream_grad(g.num_nodes, 3)
        kw = {"norm": L.rgcn_edge_norm(g, "mean")} if model == "rgcn" else {}
        ref_out, _ = L.forward(model, g, inp, **kw)
        ref = L.backward(model, g, inp, G, **kw)
        out, grads = OG.forward_backward(model, g, inp, G, **kw)
        assert _rel(out, ref_out) < 1e-12
        for k in ref:
            assert _rel(grads[k], ref[k]) < 1e-11, (model, k)


def test_grouped_no_self_loop_and_forward_only():
    g = config_graph("tiny", seed=2, scale=0.2)
    inp = layer_inputs("rgcn", g, 8, 8)
    norm = L.rgcn_edge_norm(g, "none")
    ref, _ = L.forward("rgcn", g, inp, norm=norm, self_loop=False)
    out, grads = OG.forward_backward("rgcn", g, inp, None, norm=norm, self_loop=False)
    assert grads == {} and _rel(out, ref) < 1e-12
