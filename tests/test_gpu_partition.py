"""§8(e) on one GPU: the destination-partitioned path, P logical ranks in one process.

Each "rank" builds the in-edge graph of its destination range (rgnn_graph_build with
dst_lo/dst_hi), runs the layer on the full X (what the NCCL all-gather delivers), and
back-propagates G masked to its own rows.  The owned output rows must equal the oracle's
rows, and the sums over ranks of dX and of every weight gradient (what reduce-scatter /
all-reduce compute) must equal the oracle's full gradients, at the north_star tolerances.
The collectives themselves are NCCL's; their host-side bookkeeping is tests/test_dist_cpu.py.
"""
import numpy as np
import pytest
import torch

from oracle import layers as L
from synth import config_graph, layer_inputs, upstream_grad
from tests.helpers import TOL, prepare, rel_err, to_device

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("model", ["rgcn", "rgcn_sym", "rgat", "hgt"])
def test_logical_partition(model, dtype, world):
    """rgcn_sym: the GCN normaliser 1/sqrt(d_out(s) d_in(d)) needs every source's out-degree over
    the whole graph, which a rank's in-edge graph does not hold (the library keeps the global one)."""
    from paper_2412_04747_b200 import Graph, Layer
    from paper_2412_04747_b200 import dist as D
    g = config_graph("aifb", seed=3)
    d = 64
    norm = "sym" if model == "rgcn_sym" else "mean"
    model = "rgcn" if model == "rgcn_sym" else model
    inp = prepare(layer_inputs(model, g, d, d), dtype)
    Gh = upstream_grad(g.num_nodes, d)
    kw = {"norm": L.rgcn_edge_norm(g, norm)} if model == "rgcn" else {}
    ref_out, _ = L.forward(model, g, inp, **kw)
    ref = L.backward(model, g, inp, Gh, **kw)
    dev = to_device(inp, dtype)
    X = dev.pop("X")
    ranges = D.partition_ranges(g.dst, g.num_nodes, world)
    out = np.zeros_like(ref_out)
    sums = {}
    for lo, hi in ranges:
        G = Graph.from_hetero(g, dst_range=(lo, hi))
        layer = Layer(G, model, d, d, dtype=dtype, norm=norm)
        o = layer.forward(X, dev)
        Gm = torch.zeros(g.num_nodes, d, dtype=torch.float32, device="cuda")
        Gm[lo:hi] = torch.tensor(Gh[lo:hi], dtype=torch.float32, device="cuda")
        gr = layer.backward(X, dev, o, Gm)
        torch.cuda.synchronize()
        out[lo:hi] = o.cpu().numpy()[lo:hi]
        for k, v in gr.items():
            sums[k] = sums.get(k, 0.0) + v.cpu().numpy().astype(np.float64)
    tol = TOL[dtype]
    errs = {"out": rel_err(out, ref_out)}
    for k, v in ref.items():
        errs[k] = rel_err(sums[k], v)
    bad = {k: e for k, e in errs.items() if not e <= tol}
    assert not bad, (model, dtype, world, errs)
