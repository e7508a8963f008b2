"""C1 graph-build reference (integer; the GPU build must match it bit for bit).

Definitions:
  etype_ptr[r]      = number of edges with rel < r          ("etype_ptr specifies the
                      offsets of each segment", §3.3.1; P:757 fig:compact_opt_opt)
  CSR (dst-major)   = edge ids stably ordered by (dst, rel, src, eid); row_ptr over dst
                      (COO->CSR preprocessing, §3.3.6; dst-keyed)
  CSC (src-major)   = edge ids ordered by (src, rel, dst, eid); col_ptr over src
  pairs             = distinct (rel, src) in ascending order ("compute and store the data
                      once for each (edge type, unique node index) pair", §3.3.2;
                      "unique_row_idx, unique_etype_ptr")
  pair_rel_ptr[r]   = number of pairs with rel < r   (unique_etype_ptr)
  pair_src[p]       = source node of pair p          (unique_row_idx)
  edge_pair[e]      = index of the pair (rel_e, src_e)
Written with numpy's lexsort / unique (library sorts), no blocking.
"""
from __future__ import annotations

from typing import Dict

import numpy as np


def build(num_nodes: int, num_rels: int, src: np.ndarray, dst: np.ndarray, rel: np.ndarray,
          compact: bool = True) -> Dict[str, np.ndarray]:
    """C1 arrays.  compact=False is vanilla materialization ("the row number is the
    edge index"): one row ("pair") per edge, rows in etype-sorted order with ties by
    (src, dst, eid), so pair_rel_ptr = etype_ptr and edge_pair is a bijection."""
    src = np.asarray(src, np.int64)
    dst = np.asarray(dst, np.int64)
    rel = np.asarray(rel, np.int64)
    e = len(src)
    eid = np.arange(e, dtype=np.int64)
    n, r = int(num_nodes), int(num_rels)

    etype_ptr = np.concatenate([[0], np.cumsum(np.bincount(rel, minlength=r))])

    # np.lexsort sorts by the LAST key first
    csr = np.lexsort((eid, src, rel, dst))
    row_ptr = np.concatenate([[0], np.cumsum(np.bincount(dst, minlength=n))])
    csc = np.lexsort((eid, dst, rel, src))
    col_ptr = np.concatenate([[0], np.cumsum(np.bincount(src, minlength=n))])

    if compact:
        key = rel * n + src
        ukey, edge_pair = np.unique(key, return_inverse=True)
        pair_rel = ukey // n
        pair_src = ukey % n
    else:
        order = np.lexsort((eid, dst, src, rel))
        edge_pair = np.empty(e, dtype=np.int64)
        edge_pair[order] = np.arange(e)
        pair_rel, pair_src = rel[order], src[order]
        ukey = order
    pair_rel_ptr = np.concatenate([[0], np.cumsum(np.bincount(pair_rel, minlength=r))])

    i32 = lambda a: np.asarray(a, np.int32)
    i64 = lambda a: np.asarray(a, np.int64)
    return {
        "etype_ptr": i64(etype_ptr),
        "row_ptr": i64(row_ptr), "csr_src": i32(src[csr]), "csr_rel": i32(rel[csr]), "csr_eid": i32(csr),
        "col_ptr": i64(col_ptr), "csc_dst": i32(dst[csc]), "csc_rel": i32(rel[csc]), "csc_eid": i32(csc),
        "pair_rel_ptr": i64(pair_rel_ptr), "pair_src": i32(pair_src), "edge_pair": i32(edge_pair.reshape(-1)),
        "csr_pair": i32(edge_pair.reshape(-1)[csr]), "csc_pair": i32(edge_pair.reshape(-1)[csc]),
        "num_pairs": np.int64(len(ukey)),
    }


def compaction_ratio(num_pairs: int, num_edges: int) -> float:
    """Entity compaction ratio = unique (src, etype) pairs / edges (§3.4.3);
    1.0 for an empty graph."""
    return 1.0 if num_edges == 0 else num_pairs / num_edges
