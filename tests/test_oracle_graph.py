"""Pins of the C1 graph-build oracle (oracle/graph.py).

* G7 golden arrays (tests/golden/g7_build.json);
* brute-force set semantics on the random-graph suite;
* CompactIndex invariants and the CSR round trip;
* empty graph compaction ratio 1.0.
"""
import json
import os

import numpy as np
import pytest

from oracle import graph as og
from synth import g7, random_small_graph, load_tsv, dump_tsv, config_graph

GOLD = os.path.join(os.path.dirname(__file__), "golden", "g7_build.json")


def test_g7_golden_arrays():
    gold = json.load(open(GOLD))
    g = g7()
    b = og.build(g.num_nodes, g.num_rels, g.src, g.dst, g.rel)
    for k, v in gold.items():
        if k.startswith("_") or k == "compaction_ratio":
            continue
        assert np.array_equal(np.asarray(b[k]).reshape(-1), np.asarray(v).reshape(-1)), k
    num, den = gold["compaction_ratio"]
    assert og.compaction_ratio(int(b["num_pairs"]), g.num_edges) == num / den


def _brute(g):
    """Pure-Python set semantics: sorted tuples, no numpy sorting."""
    E = g.num_edges
    edges = [(int(g.src[e]), int(g.dst[e]), int(g.rel[e]), e) for e in range(E)]
    csr = [e for (_, _, _, e) in sorted(edges, key=lambda t: (t[1], t[2], t[0], t[3]))]
    csc = [e for (_, _, _, e) in sorted(edges, key=lambda t: (t[0], t[2], t[1], t[3]))]
    pairs = sorted({(r, s) for (s, _, r, _) in edges})
    index = {p: i for i, p in enumerate(pairs)}
    edge_pair = [index[(r, s)] for (s, _, r, _) in edges]
    return csr, csc, pairs, edge_pair


@pytest.mark.parametrize("seed", range(200))
def test_random_suite_matches_brute_force(seed):
    g = random_small_graph(seed, allow_multi=(seed % 3 == 0))
    b = og.build(g.num_nodes, g.num_rels, g.src, g.dst, g.rel)
    csr, csc, pairs, edge_pair = _brute(g)
    assert list(b["csr_eid"]) == csr
    assert list(b["csc_eid"]) == csc
    assert int(b["num_pairs"]) == len(pairs)
    assert list(b["pair_src"]) == [s for (_, s) in pairs]
    assert list(b["edge_pair"]) == edge_pair
    # CompactIndex invariants S:33-39
    for e in range(g.num_edges):
        p = b["edge_pair"][e]
        assert b["pair_src"][p] == g.src[e]
        assert b["pair_rel_ptr"][g.rel[e]] <= p < b["pair_rel_ptr"][g.rel[e] + 1]
    for r in range(g.num_rels):
        seg = b["pair_src"][b["pair_rel_ptr"][r]:b["pair_rel_ptr"][r + 1]]
        assert np.all(np.diff(seg) > 0)
    # CSR round trip reproduces the COO multiset
    dst_of_entry = np.repeat(np.arange(g.num_nodes), np.diff(b["row_ptr"]))
    trip = sorted(zip(b["csr_src"].tolist(), dst_of_entry.tolist(), b["csr_rel"].tolist()))
    assert trip == sorted(zip(g.src.tolist(), g.dst.tolist(), g.rel.tolist()))
    # etype_ptr: edges of type t counted
    assert list(b["etype_ptr"]) == [int(np.sum(g.rel < r)) for r in range(g.num_rels + 1)]


def test_empty_graph_ratio_is_one():
    g = load_tsv("H 1 2\nN 4\n")
    b = og.build(g.num_nodes, g.num_rels, g.src, g.dst, g.rel)
    assert int(b["num_pairs"]) == 0
    assert og.compaction_ratio(0, 0) == 1.0
    assert list(b["row_ptr"]) == [0] * 5


def test_tsv_errors_and_roundtrip():
    with pytest.raises(ValueError, match="line 3"):
        load_tsv("H 2 2\nN 3 2\nE 0 9 0\n")
    with pytest.raises(ValueError, match="duplicate header"):
        load_tsv("H 1 1\nH 1 1\n")
    g = g7()
    g2 = load_tsv(dump_tsv(g))
    assert np.array_equal(g.src, g2.src) and np.array_equal(g.rel, g2.rel)


def test_star_and_distinct_pairs():
    # one source, k same-type edges -> one pair
    g = load_tsv("H 1 1\nN 5\n" + "".join(f"E 0 {d} 0\n" for d in range(1, 5)))
    assert int(og.build(5, 1, g.src, g.dst, g.rel)["num_pairs"]) == 1
    # every (rel, src) distinct -> bijection
    g = load_tsv("H 1 2\nN 4\nE 0 1 0\nE 1 2 0\nE 0 3 1\n")
    b = og.build(4, 2, g.src, g.dst, g.rel)
    assert int(b["num_pairs"]) == 3 and sorted(b["edge_pair"]) == [0, 1, 2]


def test_generator_deterministic_and_infeasible():
    a = config_graph("tiny", seed=1)
    b = config_graph("tiny", seed=1)
    assert np.array_equal(a.src, b.src) and np.array_equal(a.dst, b.dst) and np.array_equal(a.rel, b.rel)
    key = (a.src.astype(np.int64) * a.num_nodes + a.dst) * a.num_rels + a.rel
    assert len(np.unique(key)) == a.num_edges == 10_000
    from synth.graphs import synth_heterograph
    with pytest.raises(ValueError, match="infeasible"):
        synth_heterograph([2, 2], [(0, 1)], rel_sizes=[5])


def test_generator_compaction_calibration():
    # D1 calibration: AM-shaped a_src=0.3 gives ratio near the paper's 0.57;
    # checked on a 1/20 scale draw (ratio is roughly scale-free for fixed degree).
    g = config_graph("am", seed=1, scale=0.05)
    b = og.build(g.num_nodes, g.num_rels, g.src, g.dst, g.rel)
    ratio = og.compaction_ratio(int(b["num_pairs"]), g.num_edges)
    assert 0.45 < ratio < 0.70, ratio


@pytest.mark.parametrize("seed", range(40))
def test_vanilla_build_matches_brute_force(seed):
    """Vanilla materialization: one row per edge, rows ordered by (rel, src, dst, eid)."""
    g = random_small_graph(seed, allow_multi=(seed % 3 == 0))
    b = og.build(g.num_nodes, g.num_rels, g.src, g.dst, g.rel, compact=False)
    rows = sorted(range(g.num_edges), key=lambda e: (int(g.rel[e]), int(g.src[e]), int(g.dst[e]), e))
    assert int(b["num_pairs"]) == g.num_edges
    assert list(b["pair_src"]) == [int(g.src[e]) for e in rows]
    assert list(b["pair_rel_ptr"]) == list(b["etype_ptr"])
    assert sorted(b["edge_pair"].tolist()) == list(range(g.num_edges))
    for k, e in enumerate(rows):
        assert b["edge_pair"][e] == k


def test_vanilla_g7_seven_rows():
    g = g7()
    b = og.build(g.num_nodes, g.num_rels, g.src, g.dst, g.rel, compact=False)
    assert int(b["num_pairs"]) == 7   # "the materialized tensor involves seven rows"
