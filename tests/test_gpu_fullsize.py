"""Parity at BASELINE.json's full size, in bench.py's launch configuration
(HGT, hidden 64, bf16 tensor-core path, ogbn-mag-shaped graph: 1.94M nodes,
21.1M edges), against the fp64 oracle on sampled outputs:

* forward: output rows of sampled destinations (incl. the heaviest, split rows)
  vs the oracle on their in-edge subgraph (exact: out_v depends only on in(v));
* backward: the full backward with the upstream gradient masked to a sampled
  destination set D vs the oracle on the in-edge subgraph of D with the same
  masked gradient; every gradient (dX of all nodes, every weight) is exact under
  this decomposition (oracle/sample.py, pinned in test_oracle_layers.py).
"""
import numpy as np
import pytest
import torch

from oracle import layers as L
from oracle import sample as S
from synth import config_graph, layer_inputs, upstream_grad
from tests.helpers import TOL, prepare, rel_err, to_device

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mag():
    g = config_graph("mag", seed=1)
    inp = prepare(layer_inputs("hgt", g, 64, 64), "bf16")
    Gh = upstream_grad(g.num_nodes, 64)
    return g, inp, Gh


def _sample_dsts(g, n, seed):
    deg = np.bincount(g.dst, minlength=g.num_nodes)
    rng = np.random.default_rng(seed)
    heavy = np.argsort(-deg)[:2]                       # split rows (> 1024 in-edges)
    mid = rng.choice(np.nonzero((deg > 64) & (deg <= 1024))[0], size=8, replace=False)
    light = rng.choice(np.nonzero((deg >= 1) & (deg <= 64))[0], size=n, replace=False)
    empty = rng.choice(np.nonzero(deg == 0)[0], size=2, replace=False)
    return np.unique(np.concatenate([heavy, mid, light, empty]))


def test_mag_hgt_bf16_fullsize(mag):
    from paper_2412_04747_b200 import Graph, Layer
    g, inp, Gh = mag
    G = Graph.from_hetero(g)
    layer = Layer(G, "hgt", 64, 64, dtype="bf16")
    dev = to_device(inp, "bf16")
    X = dev.pop("X")
    out = layer.forward(X, dev)

    # ---- forward on sampled destinations
    D = _sample_dsts(g, 200, seed=0)
    _, eids = S.in_edge_subgraph(g, D)
    sub, nodes = S.compact_subgraph(g, eids)
    loc = dict(inp, X=inp["X"][nodes])
    ref_out, _ = L.forward("hgt", sub, loc)
    pos = np.searchsorted(nodes, D)
    present = (pos < len(nodes)) & (nodes[np.minimum(pos, len(nodes) - 1)] == D)
    got = out.cpu().numpy()
    ref_rows = np.zeros((len(D), 64))
    ref_rows[present] = ref_out[pos[present]]
    assert rel_err(got[D], ref_rows) <= TOL["bf16"]

    # ---- backward with G masked to D (exact decomposition over destinations)
    Gm = S.masked_grad(Gh, D)
    grads = layer.backward(X, dev, out, torch.tensor(Gm, dtype=torch.float32, device="cuda"))
    torch.cuda.synchronize()
    ref = L.backward("hgt", sub, loc, Gm[nodes])
    dX_ref = np.zeros((g.num_nodes, 64))
    dX_ref[nodes] = ref.pop("dX")
    errs = {"dX": rel_err(grads["dX"].cpu().numpy(), dX_ref)}
    for k, v in ref.items():
        errs[k] = rel_err(grads[k].cpu().numpy(), v)
    assert all(e <= TOL["bf16"] for e in errs.values()), errs
