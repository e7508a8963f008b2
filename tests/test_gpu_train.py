"""F4 training-step parity: librgnn (C-ABI) vs the fp64 oracle (oracle/train.py).

  * rgnn_nll_loss: loss and dL/dlogits vs oracle.train.nll_loss (fp32 kernel, <= 1e-5), ragged row
    counts, widths 1..1024, unlabelled rows; device-side error report (NaN) for a label >= c or a
    wrong num_labeled; deterministic (bitwise-equal reruns)
  * rgnn_relu_forward / backward: bit-exact (max(h, 0) and its bf16 RNE rounding are exact
    operations), ragged lengths
  * rgnn_sgd_update: master vs fp64 theta - lr g (<= 1e-6), bf16 shadow bit-exact to master's RNE
  * 2-layer step (RGCN / RGAT / HGT, f32 and bf16): loss, every layer's weight gradients and the
    updated weights vs oracle.train.train_step.  f32: 1e-4 (north_star).  bf16: the loss and every
    gradient at max(2e-2, 3 S), S = the oracle's own relative change of that gradient when every
    bf16-stored input (X, all weights) is perturbed by a seeded +-2^-9 relative (one bf16 rounding,
    DESIGN.md b16).  The first layer's weight gradients of a stacked bf16 step are ill-conditioned
    (S reaches 0.05 for HGT: softmax-backward cancellations, and ReLU masks that flip for |h_1| at
    the rounding level), so no bf16 implementation meets a flat 2e-2 there; a single bf16 layer
    does (tests/test_gpu_layers.py), and the f32 step checks the same chain at 1e-4.
"""
import numpy as np
import pytest
import torch

from oracle import train as OT
from synth import config_graph, random_labels, round_bf16, stack_inputs
from tests.helpers import TOL, prepare, rel_err

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,c", [(1, 1), (37, 4), (1001, 33), (5000, 64), (777, 100), (129, 1024), (3, 64), (1, 64),
                                 (513, 128), (77, 256), (100003, 64)])
def test_nll_loss(n, c):
    from paper_2412_04747_b200 import NllLoss
    rng = np.random.default_rng(n + c)
    z = rng.normal(scale=2.0, size=(n, c)).astype(np.float32)
    y = rng.integers(-1, c, size=n).astype(np.int32)
    ref_loss, ref_grad = OT.nll_loss(z.astype(np.float64), y)
    nl = int(((y >= 0) & (y < c)).sum())
    f = NllLoss(n, c)
    dz = torch.empty(n, c, device="cuda")
    zt, yt = torch.tensor(z, device="cuda"), torch.tensor(y, device="cuda")
    loss = f(zt, yt, nl, dlogits=dz).item()
    assert abs(loss - ref_loss) <= 1e-5 * max(1.0, abs(ref_loss))
    assert rel_err(dz.cpu().numpy(), ref_grad) <= 1e-5 if nl else not dz.cpu().numpy().any()
    # deterministic
    dz2 = torch.empty_like(dz)
    assert f(zt, yt, nl, dlogits=dz2).item() == loss
    assert torch.equal(dz, dz2)
    # loss only
    assert f(zt, yt, nl).item() == loss


def test_nll_errors():
    from paper_2412_04747_b200 import NllLoss, RGNNError
    z = torch.zeros(10, 8, device="cuda")
    y = torch.arange(10, dtype=torch.int32, device="cuda") % 8
    f = NllLoss(10, 8)
    assert abs(f(z, y, 10).item() - np.log(8)) < 1e-6
    assert np.isnan(f(z, y, 9).item())            # wrong labelled-row count
    y[3] = 8
    assert np.isnan(f(z, y, 10).item())           # label out of range
    assert f(z, torch.full((10,), -1, dtype=torch.int32, device="cuda"), 0).item() == 0.0
    with pytest.raises(RGNNError):
        NllLoss(10, 2000)
    e = NllLoss(0, 8)
    assert e(torch.zeros(0, 8, device="cuda"), torch.zeros(0, dtype=torch.int32, device="cuda"), 0).item() == 0.0


@pytest.mark.parametrize("n", [1, 7, 4096, 100003])
def test_relu(n):
    from paper_2412_04747_b200 import rgnn
    h = torch.tensor(np.random.default_rng(n).normal(size=n).astype(np.float32), device="cuda")
    h[: min(n, 3)] = 0.0
    for dt in (torch.float32, torch.bfloat16):
        a = rgnn.relu_forward(h, dtype=dt)
        assert torch.equal(a, torch.clamp(h, min=0).to(dt))
    da = torch.tensor(np.random.default_rng(n + 1).normal(size=n).astype(np.float32), device="cuda")
    dh = rgnn.relu_backward(h, da)
    assert torch.equal(dh, torch.where(h > 0, da, torch.zeros_like(da)))
    rgnn.relu_backward(h, da, out=da)  # in place
    assert torch.equal(da, dh)


def test_sgd_update():
    from paper_2412_04747_b200 import rgnn
    rng = np.random.default_rng(0)
    sizes = [1, 5, 64, 4099, 535 * 64 * 64] + [3] * 40      # > 32 tensors: two launches
    ms = [rng.normal(size=s) for s in sizes]
    gs = [rng.normal(size=s) for s in sizes]
    lr = 0.05
    for sdt in (torch.float32, torch.bfloat16):
        mt = [torch.tensor(m.astype(np.float32), device="cuda") for m in ms]
        gt = [torch.tensor(g.astype(np.float32), device="cuda") for g in gs]
        sh = [torch.empty(s, dtype=sdt, device="cuda") if i % 2 == 0 else None for i, s in enumerate(sizes)]
        rgnn.sgd_update(list(zip(mt, gt, sh)), lr, shadow_dtype=sdt)
        for m, g, t, s in zip(ms, gs, mt, sh):
            ref = m.astype(np.float32).astype(np.float64) - lr * g.astype(np.float32).astype(np.float64)
            assert rel_err(t.cpu().numpy(), ref) <= 1e-6
            if s is not None:
                assert torch.equal(s, t.to(sdt))


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("model,graph,scale", [("rgat", "aifb", 1.0), ("hgt", "tiny", 0.5), ("rgcn", "tiny", 0.5),
                                               ("rgat", "bgs", 0.05)])
def test_two_layer_step(model, graph, scale, dtype):
    from paper_2412_04747_b200 import Graph, Stack
    g = config_graph(graph, seed=1, scale=scale)
    d = 64
    ps = stack_inputs(model, g, d, 2)
    X = ps[0].pop("X")
    ps = [prepare(p, dtype) for p in ps]
    X = prepare({"X": X}, dtype)["X"]
    y = random_labels(g.num_nodes, d, seed=5, labelled_frac=0.8)
    lr = 0.1
    trained = OT_TRAINED[model]
    ref_loss, ref_grads, ref_new = OT.train_step(model, g, X, ps, y, lr, trained,
                                                 act_round=round_bf16 if dtype == "bf16" else None)

    G = Graph.from_hetero(g)
    st = Stack(G, model, d, [{k: torch.tensor(v) for k, v in p.items()} for p in ps], dtype=dtype)
    Xd = torch.tensor(X.astype(np.float32), device="cuda").to(st.td)
    yd = torch.tensor(y, device="cuda")
    loss = st.train_step(Xd, yd, int((y >= 0).sum()), lr).item()
    torch.cuda.synchronize()
    tols = {}
    if dtype == "bf16":
        # gradients that are ill-conditioned under one bf16 rounding of the inputs (DESIGN.md b16:
        # the oracle's own relative change S under a 2^-9 perturbation exceeds 1e-2, e.g. S = 0.11
        # for layer 2's da on the BGS shape) get max(2e-2, 2 S) in layer 2 and max(2e-2, 3 S) in
        # layer 1 (whose input gradient has passed through layer 2's backward and a ReLU mask);
        # the loss and every gradient with S <= 1e-2 are held to the flat 2e-2
        S = bf16_sensitivity(model, g, X, ps, y, trained)
        tols = {k: max(TOL[dtype], (3 if k.startswith("L0.") else 2) * v) for k, v in S.items() if k != "loss"}
    tol_of = lambda k: tols.get(k, TOL[dtype])  # noqa: E731
    assert abs(loss - ref_loss) <= tol_of("loss") * abs(ref_loss), (loss, ref_loss)
    errs = {}
    for i in range(2):
        for k in trained:
            errs[f"L{i}.d{k}"] = rel_err(st.grads[i]["d" + k].cpu().numpy(), ref_grads[i]["d" + k])
            errs[f"L{i}.{k}"] = rel_err(st.master[i][k].cpu().numpy(), ref_new[i][k])
    bad = {k: (e, tol_of(k)) for k, e in errs.items() if not e <= tol_of(k)}
    assert not bad, (bad, errs)
    # the layer-dtype copies the next step reads were refreshed from the updated masters
    for i in range(2):
        for k in trained:
            assert torch.equal(st.w[i][k], st.master[i][k].to(st.td))


def bf16_sensitivity(model, g, X, ps, y, trained, eps=2.0 ** -9, seeds=(7, 8)):
    """Relative change of the oracle's loss and gradients (keys "loss", "L{i}.d{k}") when X and every
    weight are multiplied by 1 + eps U(-1, 1) (seeded): the conditioning of each output under one
    bf16 rounding of the inputs.  Oracle only; max over the seeds."""
    l0, g0 = OT.stack_backward(model, g, X, ps, y, act_round=round_bf16)
    out = {}
    for sd in seeds:
        rng = np.random.default_rng(sd)
        jit = lambda v: v * (1.0 + eps * rng.uniform(-1.0, 1.0, np.shape(v)))  # noqa: E731
        pp = [{k: (jit(v) if k in trained else v) for k, v in p.items()} for p in ps]
        l1, g1 = OT.stack_backward(model, g, jit(X), pp, y, act_round=round_bf16)
        out["loss"] = max(out.get("loss", 0.0), abs(l1 - l0) / abs(l0))
        for i in range(len(ps)):
            for k in trained:
                key = f"L{i}.d{k}"
                out[key] = max(out.get(key, 0.0), rel_err(g1[i]["d" + k], g0[i]["d" + k]))
    return out


OT_TRAINED = {"rgcn": ("W", "W0"), "rgat": ("W", "a", "b"), "hgt": ("Wk", "Wq", "Wv", "Watt", "Wmsg")}
