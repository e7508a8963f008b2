"""Exact evaluation of sampled outputs of a large graph with the plain oracle.

TEST INFRASTRUCTURE (see oracle/__init__.py).  Uses two facts of the layer
definitions, not any GPU-side blocking:
  (1) out_v depends only on the in-edges of v (message generation on edges,
      then aggregation per destination, §3.2.1), so the in-edge
      subgraph of a destination set D reproduces out_v exactly for v in D;
  (2) L = sum_v out_v . G_v is a sum over destinations and every gradient is
      linear in G, so with G masked to rows in D (G_D) every gradient of the full
      graph equals the gradient of the in-edge subgraph of D under G_D.
"""
from __future__ import annotations

from typing import Tuple

import numpy as np

from synth.graphs import HeteroGraph


def in_edge_subgraph(g: HeteroGraph, dst_nodes: np.ndarray) -> Tuple[HeteroGraph, np.ndarray]:
    """All edges whose destination is in dst_nodes, same node id space.
    Returns (subgraph, original edge ids in subgraph order)."""
    mask = np.zeros(g.num_nodes, bool)
    mask[np.asarray(dst_nodes, np.int64)] = True
    eids = np.nonzero(mask[g.dst])[0]
    sub = HeteroGraph(g.node_type_ptr, g.num_rels, g.src[eids], g.dst[eids], g.rel[eids],
                      name=f"{g.name}[in-edges of {int(mask.sum())} dst]", rel_types=g.rel_types)
    return sub, eids


def backward_closure(g: HeteroGraph, nodes: np.ndarray) -> np.ndarray:
    """Destinations whose in-edges determine dX[u] for u in `nodes`: the nodes
    themselves plus every destination of an out-edge of theirs."""
    mask = np.zeros(g.num_nodes, bool)
    mask[np.asarray(nodes, np.int64)] = True
    d = np.unique(np.concatenate([np.asarray(nodes, np.int64), g.dst[mask[g.src]].astype(np.int64)]))
    return d


def masked_grad(G: np.ndarray, dst_nodes: np.ndarray) -> np.ndarray:
    Gm = np.zeros_like(G)
    idx = np.asarray(dst_nodes, np.int64)
    Gm[idx] = G[idx]
    return Gm


def compact_subgraph(g: HeteroGraph, eids: np.ndarray) -> Tuple[HeteroGraph, np.ndarray]:
    """The edges `eids` of g on a relabelled node set: the nodes they touch, in ascending
    original id (node types stay contiguous).  Returns (subgraph, original ids of its nodes)."""
    eids = np.asarray(eids, np.int64)
    nodes = np.unique(np.concatenate([g.src[eids], g.dst[eids]]).astype(np.int64))
    ptr = np.searchsorted(nodes, g.node_type_ptr).astype(np.int64)
    remap = lambda a: np.searchsorted(nodes, a.astype(np.int64)).astype(np.int32)
    sub = HeteroGraph(ptr, g.num_rels, remap(g.src[eids]), remap(g.dst[eids]), g.rel[eids].copy(),
                      name=f"{g.name}[{len(eids)} edges]", rel_types=g.rel_types)
    return sub, nodes
