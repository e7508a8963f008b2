"""F4: a stacked-layer training step on the C-ABI.

    layer 1 -> ReLU -> layer 2 -> ... -> NLL loss vs labels -> backward -> SGD

The paper's training measurement computes "the negative log-likelihood loss by
comparing the output with a precomputed random label tensor" (§3.4.1);
BASELINE.json's AIFB/MUTAG/BGS/AM configs stack 2 RGAT layers of width 64.
Readings (DESIGN.md b13-b15): ReLU between layers, mean NLL over labelled rows,
plain SGD on fp32 master weights with the layer-dtype copy refreshed in the same
kernel.  Argument marshalling only: every step runs in librgnn's kernels
(rgnn_layer_*, rgnn_relu_*, rgnn_nll_loss, rgnn_sgd_update).
"""
from __future__ import annotations

from typing import Dict, List, Optional, Sequence

import torch

from .rgnn import Graph, Layer, NllLoss, relu_backward, relu_forward, sgd_update

TRAINED = {"rgcn": ("W", "W0"), "rgat": ("W", "a", "b"), "hgt": ("Wk", "Wq", "Wv", "Watt", "Wmsg")}


class Stack:
    """`len(weights)` layers of one model, all of width d, bound to one graph.

    weights: per layer a dict of float32 tensors (any device; copied) with the model's
    rgnn_weights fields.  The trained ones are kept as float32 master copies; the layers
    read `self.w[i]` (the layer-dtype copies, refreshed by every SGD update)."""

    def __init__(self, graph: Graph, model: str, d: int, weights: Sequence[Dict[str, torch.Tensor]],
                 dtype: str = "bf16", heads: int = 1, tail: bool = False, **layer_kw):
        self.graph, self.model, self.d = graph, model, d
        dev = graph.device
        self.n = int(graph.info()["num_nodes"])
        self.num_layers = len(weights)
        self.layers = [Layer(graph, model, d, d, dtype=dtype, heads=heads, tail=tail, **layer_kw)
                       for _ in range(self.num_layers)]
        self.td = self.layers[0].torch_dtype
        self.trained = list(TRAINED[model]) + (["A"] if tail and model == "hgt" else [])
        if model == "rgcn" and not self.layers[0].desc.self_loop:
            self.trained.remove("W0")
        self.master: List[Dict[str, torch.Tensor]] = []
        self.w: List[Dict[str, torch.Tensor]] = []
        for p in weights:
            m, w = {}, {}
            for k, v in p.items():
                v = torch.as_tensor(v)
                if k in ("mu", "edge_norm"):
                    w[k] = v.to(device=dev, dtype=torch.float32).contiguous()
                elif k in self.trained:
                    m[k] = v.to(device=dev, dtype=torch.float32).contiguous().clone()
                    w[k] = m[k] if self.td == torch.float32 else m[k].to(self.td)
                elif k != "X":
                    w[k] = v.to(device=dev, dtype=self.td).contiguous()
            self.master.append(m)
            self.w.append(w)
        L = self.num_layers
        self.h = [torch.empty(self.n, d, dtype=torch.float32, device=dev) for _ in range(L)]
        self.a = [torch.empty(self.n, d, dtype=self.td, device=dev) for _ in range(L - 1)]
        self.dlogits = torch.empty(self.n, d, dtype=torch.float32, device=dev)
        self.grads = [{"d" + k: torch.empty_like(self.master[i][k]) for k in self.trained} for i in range(L)]
        for i in range(1, L):
            self.grads[i]["dX"] = torch.empty(self.n, d, dtype=torch.float32, device=dev)
        self.nll = NllLoss(self.n, d, device=dev)
        self._sgd = [(self.master[i][k], self.grads[i]["d" + k], None if self.td == torch.float32 else self.w[i][k])
                     for i in range(L) for k in self.trained]

    def forward(self, X: torch.Tensor) -> torch.Tensor:
        """Logits [N][d] (float32) = layer_L(ReLU(... layer_1(X)))."""
        x = X
        for i, layer in enumerate(self.layers):
            layer.forward(x, self.w[i], out=self.h[i])
            if i + 1 < self.num_layers:
                relu_forward(self.h[i], out=self.a[i])
                x = self.a[i]
        return self.h[-1]

    def backward(self, X: torch.Tensor, G: torch.Tensor) -> None:
        """Weight gradients of every layer into self.grads for dL/dlogits = G."""
        for i in range(self.num_layers - 1, -1, -1):
            xin = X if i == 0 else self.a[i - 1]
            gr = self.layers[i].backward(xin, self.w[i], self.h[i], G, need_dX=i > 0, grads=self.grads[i],
                                         need=["d" + k for k in self.trained])
            if i > 0:
                G = relu_backward(self.h[i - 1], gr["dX"], out=gr["dX"])

    def train_step(self, X: torch.Tensor, labels: torch.Tensor, num_labeled: int, lr: float) -> torch.Tensor:
        """One step: forward, NLL loss (returned on the device, value before the update),
        backward, SGD update of every trained weight."""
        logits = self.forward(X)
        loss = self.nll(logits, labels, num_labeled, dlogits=self.dlogits)
        self.backward(X, self.dlogits)
        sgd_update(self._sgd, lr, shadow_dtype=self.td)
        return loss
