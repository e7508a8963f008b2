"""Destination-partitioned multi-GPU layer; host logic + torch.distributed plumbing.

Partition: rank k owns the destination range [lo_k, hi_k), chosen so every rank
receives about E / P in-edges (contiguous prefix over the in-degree counts).  It
builds the graph of the in-edges of its range (rgnn_graph_build with dst_lo/dst_hi),
so every destination-side step (logits, softmax, aggregation) is local.  The same
ranges partition the source rows of X: rank k owns X[lo_k:hi_k].

Exchange (variant X of §8(e)):
  forward   X_full = all_gather(X_own)                    (NCCL over NVLink)
  backward  the loss decomposes over destinations, so each rank back-propagates
            G masked to its own rows; dX_own = reduce_scatter(dX_partial) and
            dW = all_reduce(dW_partial).
Exactness of the decomposition is the property pinned by
tests/test_oracle_layers.py::test_destination_decomposition.
"""
from __future__ import annotations

from typing import Dict, List, Sequence, Tuple

import numpy as np
import torch
import torch.distributed as dist


def partition_ranges(dst: np.ndarray, num_nodes: int, world: int) -> List[Tuple[int, int]]:
    """Contiguous destination ranges with ~E/world in-edges each (every node owned once).
    Cuts are placed where the running in-edge count first reaches k*E/world."""
    if world < 1:
        raise ValueError("world must be >= 1")
    deg = np.bincount(np.asarray(dst, np.int64), minlength=num_nodes)
    csum = np.concatenate([[0], np.cumsum(deg)])
    e = int(csum[-1])
    cuts = [0]
    for k in range(1, world):
        target = (k * e) // world
        c = int(np.searchsorted(csum, target, side="left"))
        c = min(max(c, cuts[-1]), num_nodes)
        cuts.append(c)
    cuts.append(num_nodes)
    return [(cuts[k], cuts[k + 1]) for k in range(world)]


def pad_ranges(ranges: Sequence[Tuple[int, int]]) -> int:
    """Row count each rank contributes to the fixed-size collectives (max range length)."""
    return max(hi - lo for lo, hi in ranges)


def all_gather_rows(local: torch.Tensor, ranges, rank: int, group=None) -> torch.Tensor:
    """Concatenate the owned row blocks of every rank (variable sizes, padded collective)."""
    world = len(ranges)
    m = pad_ranges(ranges)
    buf = torch.zeros((m,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    buf[: local.shape[0]] = local
    out = torch.empty((world * m,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, buf, group=group)
    return torch.cat([out[k * m: k * m + (hi - lo)] for k, (lo, hi) in enumerate(ranges)], dim=0)


def reduce_scatter_rows(full: torch.Tensor, ranges, rank: int, group=None) -> torch.Tensor:
    """Sum the full-size partial over ranks and return the owned rows of this rank."""
    world = len(ranges)
    m = pad_ranges(ranges)
    send = torch.zeros((world * m,) + tuple(full.shape[1:]), dtype=full.dtype, device=full.device)
    for k, (lo, hi) in enumerate(ranges):
        send[k * m: k * m + (hi - lo)] = full[lo:hi]
    recv = torch.empty((m,) + tuple(full.shape[1:]), dtype=full.dtype, device=full.device)
    dist.reduce_scatter_tensor(recv, send, group=group)
    lo, hi = ranges[rank]
    return recv[: hi - lo]


def all_reduce_grads(grads: Dict[str, torch.Tensor], keys, group=None) -> None:
    for k in keys:
        if k in grads:
            dist.all_reduce(grads[k], group=group)


def masked_rows(G: torch.Tensor, lo: int, hi: int) -> torch.Tensor:
    Gm = torch.zeros_like(G)
    Gm[lo:hi] = G[lo:hi]
    return Gm
