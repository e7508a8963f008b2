"""Diagnostic (not a test): per-tensor error of one bf16 layer under an NLL-shaped upstream gradient
vs a random one, oracle inputs only (X, W bf16-rounded; G from the oracle)."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from oracle import layers as L, train as OT
from synth import config_graph, random_labels, stack_inputs, round_bf16, upstream_grad
from tests.helpers import prepare, rel_err
from paper_2412_04747_b200 import Graph, Layer

for model, graph, scale in [("rgat", "aifb", 1.0), ("hgt", "tiny", 0.5), ("rgcn", "tiny", 0.5)]:
    g = config_graph(graph, seed=1, scale=scale)
    d = 64
    ps = stack_inputs(model, g, d, 2)
    X = round_bf16(ps[0].pop("X"))
    ps = [prepare(p, "bf16") for p in ps]
    y = random_labels(g.num_nodes, d, seed=5, labelled_frac=0.8)
    h1, _ = L.forward(model, g, dict(ps[0], X=X))
    a1 = round_bf16(OT.relu(h1))
    inp = dict(ps[1], X=a1)
    h2, _ = L.forward(model, g, inp)
    _, Gn = OT.nll_loss(h2, y)
    Gr = upstream_grad(g.num_nodes, d)
    Gm = Gr * (np.abs(Gr).max(axis=1, keepdims=True) == np.abs(Gr))  # one-hot-like random G
    G1 = Graph.from_hetero(g)
    for name, G in [("nll", Gn), ("random", Gr), ("onehot", Gm), ("nll*1e4", Gn * 1e4)]:
        ref = L.backward(model, g, inp, G)
        lay = Layer(G1, model, d, d, dtype="bf16")
        dev = {k: (torch.tensor(v, dtype=torch.float32, device="cuda") if k in ("mu",) else
                   torch.tensor(np.asarray(v, np.float32), device="cuda").to(torch.bfloat16)) for k, v in inp.items()}
        Xd = dev.pop("X")
        out = lay.forward(Xd, dev)
        gr = lay.backward(Xd, dev, out, torch.tensor(G, dtype=torch.float32, device="cuda"))
        torch.cuda.synchronize()
        errs = {k: round(rel_err(gr[k].cpu().numpy(), v), 4) for k, v in ref.items()}
        print(model, name, "out", round(rel_err(out.cpu().numpy(), h2), 5), errs, flush=True)
