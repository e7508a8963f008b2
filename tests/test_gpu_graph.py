"""A0 graph build on the GPU: bit-exact against the C1 oracle (oracle/graph.py)."""
import json
import os

import numpy as np
import pytest
import torch

from oracle import graph as og
from synth import g7, random_small_graph, config_graph
from synth.graphs import HeteroGraph

pytestmark = pytest.mark.gpu

ARRAYS = ["etype_ptr", "row_ptr", "csr_src", "csr_rel", "csr_eid", "col_ptr", "csc_dst", "csc_rel", "csc_eid",
          "pair_rel_ptr", "pair_src", "edge_pair", "csr_pair", "csc_pair"]


def _check(g, dst_range=None):
    from paper_2412_04747_b200 import Graph
    G = Graph.from_hetero(g, dst_range=dst_range)
    if dst_range is None:
        sub = g
    else:
        m = (g.dst >= dst_range[0]) & (g.dst < dst_range[1])
        sub = HeteroGraph(g.node_type_ptr, g.num_rels, g.src[m], g.dst[m], g.rel[m])
    ref = og.build(sub.num_nodes, sub.num_rels, sub.src, sub.dst, sub.rel)
    info = G.info()
    assert info["num_edges"] == sub.num_edges
    assert info["num_pairs"] == int(ref["num_pairs"])
    assert info["compaction_ratio"] == og.compaction_ratio(int(ref["num_pairs"]), sub.num_edges)
    for name in ARRAYS:
        got = G.export(name).cpu().numpy().astype(np.int64)
        want = np.asarray(ref[name], np.int64)
        assert np.array_equal(got, want), name
    return G


def test_g7_bit_exact():
    G = _check(g7())
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "g7_build.json")))
    assert G.export("pair_src").cpu().tolist() == gold["pair_src"]


@pytest.mark.parametrize("seed", range(40))
def test_random_suite(seed):
    _check(random_small_graph(seed, allow_multi=(seed % 3 == 0)))


@pytest.mark.parametrize("name", ["tiny", "aifb", "mutag"])
def test_configs(name):
    _check(config_graph(name, seed=1))


def test_partition_ranges():
    g = config_graph("tiny", seed=2)
    n = g.num_nodes
    for lo, hi in [(0, n // 3), (n // 3, 2 * n // 3), (2 * n // 3, n), (5, 5)]:
        _check(g, dst_range=(lo, hi))


def test_empty_and_errors():
    from paper_2412_04747_b200 import Graph, RGNNError
    G = Graph(4, [0, 4], 2, torch.zeros(0, dtype=torch.int32), torch.zeros(0, dtype=torch.int32),
              torch.zeros(0, dtype=torch.int32))
    assert G.info()["compaction_ratio"] == 1.0 and G.info()["num_pairs"] == 0
    with pytest.raises(RGNNError, match="edge 2"):
        Graph(4, [0, 4], 2, torch.tensor([0, 1, 9]), torch.tensor([1, 2, 3]), torch.tensor([0, 0, 0]))
    with pytest.raises(RGNNError, match="edge 1"):
        Graph(4, [0, 4], 2, torch.tensor([0, 1, 2]), torch.tensor([1, 2, 3]), torch.tensor([0, 2, 0]))


@pytest.mark.slow
def test_mag_bit_exact():
    _check(config_graph("mag", seed=1))


@pytest.mark.parametrize("seed", range(12))
def test_vanilla_build_bit_exact(seed):
    """compact=0: vanilla materialization, one row per edge, bit-exact vs the oracle."""
    from paper_2412_04747_b200 import Graph
    g = random_small_graph(300 + seed, allow_multi=(seed % 2 == 0)) if seed < 10 else config_graph("tiny", seed=seed)
    G = Graph.from_hetero(g, compact=False)
    ref = og.build(g.num_nodes, g.num_rels, g.src, g.dst, g.rel, compact=False)
    assert G.info()["num_pairs"] == g.num_edges
    for name in ARRAYS:
        assert np.array_equal(G.export(name).cpu().numpy().astype(np.int64), np.asarray(ref[name], np.int64)), name
