"""The library-owned communicator (include/rgnn.h) on one GPU: a world-1 NCCL
communicator through rgnn_layer_forward / rgnn_layer_backward gives bit-for-bit the single-GPU
layer (the all-gather is a broadcast of the own rows onto themselves, the reductions sum one
term), and the argument checks tie the communicator's rows to the graph's destination range.
The multi-rank exchange schedule itself is restated and checked on CPU (tests/test_dist_cpu.py);
every step of the partitioned compute is checked by tests/test_gpu_partition.py."""
import numpy as np
import pytest
import torch

from synth import config_graph, layer_inputs, upstream_grad
from tests.helpers import prepare, to_device

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def comm_factory():
    from paper_2412_04747_b200 import rgnn
    made = []

    def make(n):
        c = rgnn.Comm(0, 1, [0, n], rgnn.comm_unique_id())
        made.append(c)
        return c
    yield make
    for c in made:
        c.close()


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("model", ["rgcn", "rgat", "hgt"])
def test_world1_comm_bit_exact(model, dtype, comm_factory):
    from paper_2412_04747_b200 import Graph, Layer
    g = config_graph("aifb", seed=2)
    d = 64
    inp = prepare(layer_inputs(model, g, d, d), dtype)
    dev = to_device(inp, dtype)
    X = dev.pop("X")
    dout = torch.tensor(upstream_grad(g.num_nodes, d), dtype=torch.float32, device="cuda")
    G = Graph.from_hetero(g)
    res = []
    for use in (False, True):
        comm = comm_factory(g.num_nodes) if use else None
        layer = Layer(G, model, d, d, dtype=dtype)
        Xb = X.clone()
        out = layer.forward(Xb, dev, comm=comm)
        grads = layer.backward(Xb, dev, out, dout, comm=comm)
        torch.cuda.synchronize()
        assert torch.equal(Xb, X)
        res.append((out.clone(), {k: v.clone() for k, v in grads.items()}))
    (o0, g0), (o1, g1) = res
    assert torch.equal(o0, o1)
    for k in g0:
        assert torch.equal(g0[k], g1[k]), k


def test_comm_range_must_match_graph(comm_factory):
    from paper_2412_04747_b200 import Graph, Layer, RGNNError
    g = config_graph("tiny", seed=1, scale=0.3)
    G = Graph.from_hetero(g, dst_range=(0, g.num_nodes // 2))
    layer = Layer(G, "hgt", 32, 32, dtype="f32")
    dev = to_device(layer_inputs("hgt", g, 32, 32), "f32")
    X = dev.pop("X")
    with pytest.raises(RGNNError, match="destination range"):
        layer.forward(X, dev, comm=comm_factory(g.num_nodes))


def test_comm_unique_ids_differ():
    from paper_2412_04747_b200 import rgnn
    a, b = rgnn.comm_unique_id(), rgnn.comm_unique_id()
    assert len(a) == rgnn.COMM_ID_BYTES and a != b
