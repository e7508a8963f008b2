"""Destination-partitioned multi-GPU layer: host logic + torch.distributed plumbing.

Partition: rank k owns the node rows [lo_k, hi_k), chosen so every rank receives about E / P
in-edges (contiguous prefix over the in-degree counts).  It builds the graph of the in-edges of
its range (rgnn_graph_build with dst_lo/dst_hi), so every destination-side step (logits, softmax,
aggregation, Q, the self-loop) is local, and the same ranges partition the rows of X, out and dX.

The exchange itself is library-owned (include/rgnn.h "communicator"): `make_comm` shares one
NCCL unique id over the torch process group (the only use of torch.distributed on the data path
is this bootstrap) and creates the rgnn communicator; rgnn_layer_forward then all-gathers X in
owner chunks on the library's stream, overlapped with the pair GEMM, and rgnn_layer_backward
reduces dX onto the owners and all-reduces the weight gradients.

`allgather_rows_reference` / `reduce_rows_reference` restate that exchange schedule with
torch.distributed (one broadcast / reduce per owner, in place) for the world-size-2 gloo tests
on CPU, which check that the per-rank decomposition reproduces the single-process oracle.
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


def node_ptr(ranges: Sequence[Tuple[int, int]]) -> List[int]:
    """[world+1] row boundaries of contiguous ranges (rgnn_comm_create's node_ptr)."""
    out = [int(ranges[0][0])] + [int(hi) for _, hi in ranges]
    if out[0] != 0 or any(ranges[k][1] != ranges[k + 1][0] for k in range(len(ranges) - 1)):
        raise ValueError("ranges must be contiguous and start at 0")
    return out


def share_unique_id(make_id, group=None) -> bytes:
    """Rank 0 draws the id (make_id()), every rank returns the same bytes (torch.distributed
    broadcast of a byte tensor; works over gloo and nccl process groups)."""
    rank = dist.get_rank(group)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    raw = make_id() if rank == 0 else None
    n = torch.tensor([len(raw) if raw is not None else 0], dtype=torch.int64, device=dev)
    dist.broadcast(n, src=0, group=group)
    buf = torch.zeros(int(n.item()), dtype=torch.uint8, device=dev)
    if rank == 0:
        buf.copy_(torch.frombuffer(bytearray(raw), dtype=torch.uint8))
    dist.broadcast(buf, src=0, group=group)
    return bytes(buf.cpu().numpy().tobytes())


def make_comm(ranges: Sequence[Tuple[int, int]], group=None):
    """The library communicator of this rank for the given row partition (collective)."""
    from .rgnn import Comm, comm_unique_id
    uid = share_unique_id(comm_unique_id, group)
    return Comm(dist.get_rank(group), dist.get_world_size(group), node_ptr(ranges), uid)


# ----------------------------------------------------------------- CPU restatement (gloo tests)
def allgather_rows_reference(rows: torch.Tensor, ranges, group=None) -> None:
    """In-place all-gather by owner: the rows of each rank are broadcast from it (the library's
    forward schedule, one broadcast per owner)."""
    for k, (lo, hi) in enumerate(ranges):
        if hi > lo:
            chunk = rows[lo:hi].contiguous()
            dist.broadcast(chunk, src=k, group=group)
            rows[lo:hi] = chunk


def reduce_rows_reference(partial: torch.Tensor, ranges, group=None) -> None:
    """In-place reduce onto the owners: after the call rank k's rows [lo_k, hi_k) hold the sum over
    ranks (the library's backward schedule, one reduce per owner)."""
    for k, (lo, hi) in enumerate(ranges):
        if hi > lo:
            chunk = partial[lo:hi].contiguous()
            dist.reduce(chunk, dst=k, group=group)
            if dist.get_rank(group) == k:
                partial[lo:hi] = chunk


def all_reduce_grads(grads: Dict[str, torch.Tensor], keys, group=None) -> None:
    for k in keys:
        if k in grads:
            dist.all_reduce(grads[k], group=group)
