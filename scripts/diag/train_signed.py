"""Diagnostic: bf16 HGT layer on sign-structured inputs, single layer, random G vs the chain G."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from oracle import layers as L, train as OT
from synth import config_graph, random_labels, stack_inputs, round_bf16, upstream_grad
from synth.inputs import sign_structured
from tests.helpers import prepare, rel_err
from paper_2412_04747_b200 import Graph, Layer, Stack

model = sys.argv[1] if len(sys.argv) > 1 else "hgt"
g = config_graph("tiny", seed=1, scale=0.5)
d = 64
ps = stack_inputs(model, g, d, 2)
X = ps[0].pop("X")
ps[0], X = sign_structured(ps[0], model, X)
X = round_bf16(X)
ps = [prepare(p, "bf16") for p in ps]
y = random_labels(g.num_nodes, d, seed=5, labelled_frac=0.8)
h1, _ = L.forward(model, g, dict(ps[0], X=X))
a1 = round_bf16(OT.relu(h1))
h2, _ = L.forward(model, g, dict(ps[1], X=a1))
_, Gn = OT.nll_loss(h2, y)
G1 = L.backward(model, g, dict(ps[1], X=a1), Gn)["dX"] * (h1 > 0)
Gr = upstream_grad(g.num_nodes, d)
G = Graph.from_hetero(g)
for name, GG in [("random", Gr), ("chainG1", G1), ("chainG1*1e4", G1 * 1e4)]:
    inp = dict(ps[0], X=X)
    ref = L.backward(model, g, inp, GG)
    lay = Layer(G, model, d, d, dtype="bf16")
    dev = {k: (torch.tensor(v, dtype=torch.float32, device="cuda") if k == "mu" else
               torch.tensor(np.asarray(v, np.float32), device="cuda").to(torch.bfloat16)) for k, v in inp.items()}
    Xd = dev.pop("X")
    out = lay.forward(Xd, dev)
    gr = lay.backward(Xd, dev, out, torch.tensor(GG, dtype=torch.float32, device="cuda"))
    torch.cuda.synchronize()
    print(name, "out", round(rel_err(out.cpu().numpy(), h1), 5),
          {k: round(rel_err(gr[k].cpu().numpy(), v), 4) for k, v in ref.items()}, flush=True)
# the full stack
st = Stack(G, model, d, [{k: torch.tensor(v) for k, v in p.items()} for p in ps], dtype="bf16")
loss = st.train_step(torch.tensor(X.astype(np.float32), device="cuda").to(torch.bfloat16), torch.tensor(y, device="cuda"),
                     int((y >= 0).sum()), 0.0).item()
ref_loss, ref_grads = OT.stack_backward(model, g, X, ps, y, act_round=round_bf16)
print("stack loss", loss, ref_loss, "h1", rel_err(st.h[0].cpu().numpy(), h1), "h2", rel_err(st.h[1].cpu().numpy(), h2))
print("dlogits", rel_err(st.dlogits.cpu().numpy(), Gn))
for i in range(2):
    print("layer", i, {k: round(rel_err(st.grads[i][k].cpu().numpy(), ref_grads[i][k]), 4) for k in ref_grads[i]})
