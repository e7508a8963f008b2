"""World-size-2 gloo test of the destination-partitioned multi-GPU bookkeeping
(paper_2412_04747_b200/dist.py) on CPU: partition ranges, all-gather of owned
rows, masked-G backward, reduce-scatter of dX and all-reduce of dW reproduce
the single-process oracle exactly (the per-rank compute is the oracle on the
rank's in-edge subgraph, i.e. what each GPU computes)."""
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
        # forward exchange: all-gather the owned source rows of X
        X_full = D.all_gather_rows(torch.from_numpy(inp["X"][lo:hi]), ranges, rank).numpy()
        assert np.array_equal(X_full, inp["X"])
        sub, eids = S.in_edge_subgraph(g, np.arange(lo, hi))
        kw = {"norm": L.rgcn_edge_norm(g, "mean")[eids]} if model == "rgcn" else {}
        local = dict(inp, X=X_full)
        out, _ = L.forward(model, sub, local, **kw)
        out_full = D.all_gather_rows(torch.from_numpy(out[lo:hi]), ranges, rank).numpy()
        grads = L.backward(model, sub, local, S.masked_grad(Gh, np.arange(lo, hi)), **kw)
        dX_own = D.reduce_scatter_rows(torch.from_numpy(grads.pop("dX")), ranges, rank)
        dX_full = D.all_gather_rows(dX_own, ranges, rank).numpy()
        tg = {k: torch.from_numpy(v) for k, v in grads.items()}
        D.all_reduce_grads(tg, list(tg))
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
