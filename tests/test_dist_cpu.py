"""World-size-2 gloo test of the destination-partitioned multi-GPU bookkeeping
(paper_2412_04747_b200/dist.py) on CPU: partition ranges, the library's exchange schedule
restated with torch.distributed (in-place all-gather of X by owner broadcasts, reduce of the
partial dX onto the owners, all-reduce of dW), and the owned-rows-only dout reproduce the
single-process oracle exactly (the per-rank compute is the oracle on the rank's in-edge
subgraph, i.e. what each GPU computes); plus the NCCL unique-id bootstrap over the process
group (the only torch.distributed call the GPU path makes)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import layers as L
from oracle import sample as S
from synth import config_graph, layer_inputs, upstream_grad


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, model, q):
    from paper_2412_04747_b200 import dist as D
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = config_graph("tiny", seed=11, scale=0.3)
        inp = layer_inputs(model, g, 8, 8)
        Gh = upstream_grad(g.num_nodes, 8)
        ranges = D.partition_ranges(g.dst, g.num_nodes, world)
        lo, hi = ranges[rank]
        # forward exchange: rows of other ranks are garbage until the owner broadcasts arrive
        X = torch.full(inp["X"].shape, float("nan"), dtype=torch.float64)
        X[lo:hi] = torch.from_numpy(inp["X"][lo:hi])
        D.allgather_rows_reference(X, ranges)
        X_full = X.numpy()
        assert np.array_equal(X_full, inp["X"])
        sub, eids = S.in_edge_subgraph(g, np.arange(lo, hi))
        kw = {"norm": L.rgcn_edge_norm(g, "mean")[eids]} if model == "rgcn" else {}
        local = dict(inp, X=X_full)
        out, _ = L.forward(model, sub, local, **kw)
        out_t = torch.from_numpy(np.ascontiguousarray(out))
        D.allgather_rows_reference(out_t, ranges)   # only to compare the whole output on rank 0
        out_full = out_t.numpy()
        # dout: only the owned rows are read (the rest is never touched on a rank)
        Gown = np.full_like(Gh, np.nan)
        Gown[lo:hi] = Gh[lo:hi]
        grads = L.backward(model, sub, local, np.where(np.isnan(Gown), 0.0, Gown), **kw)
        dX = torch.from_numpy(np.ascontiguousarray(grads.pop("dX")))
        D.reduce_rows_reference(dX, ranges)
        D.allgather_rows_reference(dX, ranges)      # only to compare the whole dX on rank 0
        dX_full = dX.numpy()
        tg = {k: torch.from_numpy(v) for k, v in grads.items()}
        D.all_reduce_grads(tg, list(tg))
        # the NCCL-id bootstrap: rank 0's bytes reach every rank unchanged
        uid = D.share_unique_id(lambda: bytes(range(128)))
        assert uid == bytes(range(128))
        if rank == 0:
            ref_out, _ = L.forward(model, g, inp)
            ref = L.backward(model, g, inp, Gh)
            err = {"out": float(np.max(np.abs(out_full - ref_out))), "dX": float(np.max(np.abs(dX_full - ref["dX"])))}
            for k, v in tg.items():
                err[k] = float(np.max(np.abs(v.numpy() - ref[k])))
            q.put((ranges, err))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("model", ["rgcn", "rgat", "hgt"])
def test_two_rank_partition_matches_oracle(model):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, model, q)) for r in range(2)]
    for p in procs:
        p.start()
    ranges, err = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ranges[0][0] == 0 and ranges[-1][1] > ranges[0][1]
    assert max(err.values()) < 1e-12, err


def test_node_ptr():
    from paper_2412_04747_b200.dist import node_ptr
    assert node_ptr([(0, 3), (3, 3), (3, 10)]) == [0, 3, 3, 10]
    with pytest.raises(ValueError):
        node_ptr([(0, 3), (4, 10)])


def test_partition_ranges_balance():
    from paper_2412_04747_b200.dist import partition_ranges
    g = config_graph("tiny", seed=1)
    for world in (1, 2, 3, 8):
        r = partition_ranges(g.dst, g.num_nodes, world)
        assert r[0][0] == 0 and r[-1][1] == g.num_nodes
        assert all(r[k][1] == r[k + 1][0] for k in range(world - 1))
        deg = np.bincount(g.dst, minlength=g.num_nodes)
        loads = [deg[lo:hi].sum() for lo, hi in r]
        assert max(loads) <= g.num_edges / world + deg.max()
