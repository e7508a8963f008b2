"""Plain fp64 per-edge ("vanilla materialization") definitions of one RGNN layer.

TEST INFRASTRUCTURE (see oracle/__init__.py).  Everything is evaluated once per
EDGE, exactly as the paper writes the layer, with no compaction and no
linear-operator reordering: compaction and reordering are exact rewrites
("eliminate repetitive identical computations", §3.3.2; reordering is
associativity of linear operators, §3.3.2), so the GPU's compact,
reordered evaluation must agree with this one up to rounding.

Library primitives used as steps: numpy matmul (per relation / per node type),
np.add.at / np.maximum.at for segment sums / maxima by destination or source.

Notation: edge e = (s_e, d_e, r_e); tau(n) node type; in(v) = {e : d_e = v};
loss L = sum(out * G) so G = dL/dout (reading g12).

Readings (restated in DESIGN.md): g1 RGCN norm, g2 sigma =
identity, g3 self-loop only for RGCN, g4 RGAT message = h_s W_r, g5 softmax over
all incoming edges of v across relations, g6 LeakyReLU slope 0.2 with
derivative slope at z = 0, g7 HGT formula, g8 one head, g9 max-shifted
softmax, g10 empty rows give zero aggregation.
"""
from __future__ import annotations

from typing import Dict, Tuple

import numpy as np

from synth.graphs import HeteroGraph


# ----------------------------------------------------------------- primitives
def typed_matmul(rows: np.ndarray, W: np.ndarray, types: np.ndarray, transpose: bool = False) -> np.ndarray:
    """Row i -> rows[i] @ W[types[i]]  (or @ W[types[i]].T).  The typed linear of the
    GEMM template Y = X[G] x W[T] (§3.3.3), one row at a time in meaning."""
    d_out = W.shape[1] if transpose else W.shape[2]
    out = np.zeros((rows.shape[0], d_out))
    for t in np.unique(types):
        m = types == t
        Wt = W[t].T if transpose else W[t]
        out[m] = rows[m] @ Wt
    return out


def segment_sum(values: np.ndarray, seg: np.ndarray, n: int) -> np.ndarray:
    out = np.zeros((n,) + values.shape[1:])
    np.add.at(out, seg, values)
    return out


def typed_outer_sum(A: np.ndarray, B: np.ndarray, types: np.ndarray, num_types: int) -> np.ndarray:
    """dW[t] = sum_{i: types[i]=t} A[i]^T B[i]  (weight gradient of a typed linear)."""
    out = np.zeros((num_types, A.shape[1], B.shape[1]))
    for t in range(num_types):
        m = types == t
        if m.any():
            out[t] = A[m].T @ B[m]
    return out


def leaky_relu(z: np.ndarray, slope: float) -> np.ndarray:
    """sigma of RGAT is a leaky ReLU (P:563 fig:rgat_layer caption); slope reading g6."""
    return np.where(z > 0, z, slope * z)


def edge_softmax(logits: np.ndarray, dst: np.ndarray, n: int) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    """edge_softmax of lst:ir_example: att = exp(att) / sum over n.incoming_edges().
    Max-shifted (reading g9; mathematically identical).  Returns (alpha, m, s)."""
    m = np.full(n, -np.inf)
    np.maximum.at(m, dst, logits)
    ex = np.exp(logits - m[dst])
    s = np.zeros(n)
    np.add.at(s, dst, ex)
    return ex / s[dst], m, s


def edge_softmax_backward(alpha: np.ndarray, dalpha: np.ndarray, dst: np.ndarray, n: int) -> np.ndarray:
    """dl_e = alpha_e (dalpha_e - sum_{e' in in(d_e)} alpha_e' dalpha_e')  (softmax Jacobian)."""
    row = np.zeros(n)
    np.add.at(row, dst, alpha * dalpha)
    return alpha * (dalpha - row[dst])


def rgcn_edge_norm(g: HeteroGraph, kind: str = "mean") -> np.ndarray:
    """Multiplier 1/c_{v,r} of Eq. 3.1 per edge (reading g1).
    'mean': 1/|{e' in in(d_e): r_e' = r_e}|  (mean over the relation's in-neighbours)
    'sym' : 1/sqrt(d_out(s_e) * d_in(d_e))   (GCN A*)
    'none': 1."""
    e = g.num_edges
    if kind == "none":
        return np.ones(e)
    if kind == "mean":
        key = g.dst.astype(np.int64) * g.num_rels + g.rel
        _, inv, cnt = np.unique(key, return_inverse=True, return_counts=True)
        return 1.0 / cnt[inv.reshape(-1)]
    if kind == "sym":
        dout = np.bincount(g.src, minlength=g.num_nodes).astype(np.float64)
        din = np.bincount(g.dst, minlength=g.num_nodes).astype(np.float64)
        return 1.0 / (np.sqrt(dout[g.src]) * np.sqrt(din[g.dst]))
    raise ValueError(kind)


# ----------------------------------------------------------------- RGCN (C3)
def rgcn_forward(g: HeteroGraph, X, W, W0, norm, self_loop: bool = True):
    """Eq. 3.1: out_v = h_v W_0 + sum_r sum_{u in N_v^r} (1/c_{v,r}) h_u W_r, sigma = id (g2)."""
    msg = typed_matmul(X[g.src], W, g.rel)                       # h_u W_r per edge
    out = segment_sum(norm[:, None] * msg, g.dst, g.num_nodes)   # node aggregation
    if self_loop:
        out = out + X @ W0                                        # virtual self-loop
    return out, {"msg": msg}


def rgcn_backward(g: HeteroGraph, X, W, W0, norm, G, self_loop: bool = True) -> Dict[str, np.ndarray]:
    dmsg = norm[:, None] * G[g.dst]
    dX = segment_sum(typed_matmul(dmsg, W, g.rel, transpose=True), g.src, g.num_nodes)
    dW = typed_outer_sum(X[g.src], dmsg, g.rel, g.num_rels)
    grads = {"dX": dX, "dW": dW}
    if self_loop:
        grads["dX"] = dX + G @ W0.T
        grads["dW0"] = X.T @ G
    return grads


# ----------------------------------------------------------------- RGAT (C4)
def rgat_forward(g: HeteroGraph, X, W, a, b, slope: float = 0.2):
    """lst:ir_example + message h_s W_r (g4) + attention-weighted sum:
         hs = h_src W_r ; atts = hs . w_s[r] ; ht = h_dst W_r ; attt = ht . w_t[r]
         att = leakyrelu(atts + attt) ; alpha = edge_softmax ; out_v = sum alpha_e hs_e."""
    n = g.num_nodes
    hs = typed_matmul(X[g.src], W, g.rel)
    ht = typed_matmul(X[g.dst], W, g.rel)
    z = np.sum(hs * a[g.rel], axis=1) + np.sum(ht * b[g.rel], axis=1)
    l = leaky_relu(z, slope)
    alpha, m, s = edge_softmax(l, g.dst, n)
    out = segment_sum(alpha[:, None] * hs, g.dst, n)
    return out, {"hs": hs, "ht": ht, "z": z, "logit": l, "alpha": alpha, "m": m, "s": s}


def rgat_backward(g: HeteroGraph, X, W, a, b, G, slope: float = 0.2) -> Dict[str, np.ndarray]:
    n, R = g.num_nodes, g.num_rels
    _, c = rgat_forward(g, X, W, a, b, slope)
    hs, ht, z, alpha = c["hs"], c["ht"], c["z"], c["alpha"]
    Gd = G[g.dst]
    dalpha = np.sum(Gd * hs, axis=1)
    dl = edge_softmax_backward(alpha, dalpha, g.dst, n)
    dz = dl * np.where(z > 0, 1.0, slope)
    dhs = alpha[:, None] * Gd + dz[:, None] * a[g.rel]
    dht = dz[:, None] * b[g.rel]
    da = segment_sum(dz[:, None] * hs, g.rel, R)
    db = segment_sum(dz[:, None] * ht, g.rel, R)
    dW = typed_outer_sum(X[g.src], dhs, g.rel, R) + typed_outer_sum(X[g.dst], dht, g.rel, R)
    dX = (segment_sum(typed_matmul(dhs, W, g.rel, transpose=True), g.src, n)
          + segment_sum(typed_matmul(dht, W, g.rel, transpose=True), g.dst, n))
    return {"dX": dX, "dW": dW, "da": da, "db": db}


# ----------------------------------------------------------------- HGT (C5, reading g7)
def _heads(x: np.ndarray, heads: int) -> np.ndarray:
    """[E, d] -> [E, heads, d / heads]: head h owns the contiguous columns h*dh .. (h+1)*dh - 1."""
    return x.reshape(x.shape[0], heads, x.shape[1] // heads)


def hgt_forward(g: HeteroGraph, X, Wk, Wq, Wv, Watt, Wmsg, mu, heads: int = 1):
    """HGT message passing (reading g7 of fig:rgat_layer), H heads (the traversal
    template's head loop, algo:traversal_template P:926; reading b12: head h owns columns
    h*dh..(h+1)*dh-1 of K', q and M, dh = d_out / H):
         k = h_s Wk_tau(s) ; v = h_s Wv_tau(s) ; q = h_d Wq_tau(d)
         K'_e = k Watt_r ; M_e = v Wmsg_r ; l_{e,h} = mu_r (K'_{e,h} . q_{e,h}) / sqrt(dh)
         alpha_{.,h} = edge_softmax per head ; out_{v,h} = sum alpha_{e,h} M_{e,h}."""
    n = g.num_nodes
    tau = g.node_type_of()
    d_out = Watt.shape[2]
    dh = d_out // heads
    k = typed_matmul(X[g.src], Wk, tau[g.src])
    v = typed_matmul(X[g.src], Wv, tau[g.src])
    q = typed_matmul(X[g.dst], Wq, tau[g.dst])
    Kp = typed_matmul(k, Watt, g.rel)
    M = typed_matmul(v, Wmsg, g.rel)
    l = mu[g.rel][:, None] * np.sum(_heads(Kp, heads) * _heads(q, heads), axis=2) / np.sqrt(dh)  # [E, H]
    alpha = np.zeros_like(l)
    m = np.zeros((n, heads))
    s = np.zeros((n, heads))
    for h in range(heads):
        alpha[:, h], m[:, h], s[:, h] = edge_softmax(l[:, h], g.dst, n)
    out = segment_sum((alpha[:, :, None] * _heads(M, heads)).reshape(M.shape), g.dst, n)
    if heads == 1:
        l, alpha, m, s = l[:, 0], alpha[:, 0], m[:, 0], s[:, 0]
    return out, {"k": k, "v": v, "q": q, "Kp": Kp, "M": M, "logit": l, "alpha": alpha, "m": m, "s": s}


def hgt_backward(g: HeteroGraph, X, Wk, Wq, Wv, Watt, Wmsg, mu, G, heads: int = 1) -> Dict[str, np.ndarray]:
    n, R, T = g.num_nodes, g.num_rels, g.num_node_types
    tau = g.node_type_of()
    d_out = Watt.shape[2]
    dh = d_out // heads
    _, c = hgt_forward(g, X, Wk, Wq, Wv, Watt, Wmsg, mu, heads)
    k, v, q, Kp, M = c["k"], c["v"], c["q"], c["Kp"], c["M"]
    alpha = c["alpha"].reshape(-1, heads)
    Gd = G[g.dst]
    dalpha = np.sum(_heads(Gd, heads) * _heads(M, heads), axis=2)  # [E, H]
    dl = np.zeros_like(dalpha)
    for h in range(heads):
        dl[:, h] = edge_softmax_backward(alpha[:, h], dalpha[:, h], g.dst, n)
    scale = mu[g.rel] / np.sqrt(dh)
    dM = (alpha[:, :, None] * _heads(Gd, heads)).reshape(Gd.shape)
    dKp = ((dl * scale[:, None])[:, :, None] * _heads(q, heads)).reshape(q.shape)
    dq = ((dl * scale[:, None])[:, :, None] * _heads(Kp, heads)).reshape(Kp.shape)
    dWmsg = typed_outer_sum(v, dM, g.rel, R)
    dWatt = typed_outer_sum(k, dKp, g.rel, R)
    dv = typed_matmul(dM, Wmsg, g.rel, transpose=True)
    dk = typed_matmul(dKp, Watt, g.rel, transpose=True)
    ts, td = tau[g.src], tau[g.dst]
    dWk = typed_outer_sum(X[g.src], dk, ts, T)
    dWv = typed_outer_sum(X[g.src], dv, ts, T)
    dWq = typed_outer_sum(X[g.dst], dq, td, T)
    dX = (segment_sum(typed_matmul(dk, Wk, ts, transpose=True) + typed_matmul(dv, Wv, ts, transpose=True), g.src, n)
          + segment_sum(typed_matmul(dq, Wq, td, transpose=True), g.dst, n))
    return {"dX": dX, "dWk": dWk, "dWq": dWq, "dWv": dWv, "dWatt": dWatt, "dWmsg": dWmsg}


# ----------------------------------------------------------------- HGT layer tail (F2, reading b12)
_erf = np.vectorize(__import__("math").erf, otypes=[float])


def gelu(x: np.ndarray) -> np.ndarray:
    """GELU(x) = x Phi(x) = x (1 + erf(x / sqrt 2)) / 2 (the exact, erf form)."""
    return 0.5 * x * (1.0 + _erf(x / np.sqrt(2.0)))


def gelu_grad(x: np.ndarray) -> np.ndarray:
    """d GELU / dx = Phi(x) + x phi(x)."""
    return 0.5 * (1.0 + _erf(x / np.sqrt(2.0))) + x * np.exp(-0.5 * x * x) / np.sqrt(2.0 * np.pi)


def hgt_tail_forward(g: HeteroGraph, h, X, A):
    """HGT's output transform (the target-type "A-linear" with a residual, reading b12):
    out_v = GELU(h_v) A_tau(v) + X_v."""
    return typed_matmul(gelu(h), A, g.node_type_of()) + X


def hgt_tail_backward(g: HeteroGraph, h, X, A, G):
    """Returns (dh, dA); the residual adds G to dX."""
    tau = g.node_type_of()
    dA = typed_outer_sum(gelu(h), G, tau, g.num_node_types)
    dh = typed_matmul(G, A, tau, transpose=True) * gelu_grad(h)
    return dh, dA


# ----------------------------------------------------------------- dispatch
PARAMS = {"rgcn": ("W", "W0"), "rgat": ("W", "a", "b"), "hgt": ("Wk", "Wq", "Wv", "Watt", "Wmsg")}


def forward(model: str, g: HeteroGraph, inp: Dict[str, np.ndarray], *, norm=None, norm_kind: str = "mean",
            self_loop: bool = True, slope: float = 0.2, heads: int = 1, tail: bool = False):
    if model == "rgcn":
        if norm is None:
            norm = rgcn_edge_norm(g, norm_kind)
        return rgcn_forward(g, inp["X"], inp["W"], inp["W0"], norm, self_loop)
    if model == "rgat":
        return rgat_forward(g, inp["X"], inp["W"], inp["a"], inp["b"], slope)
    if model == "hgt":
        h, c = hgt_forward(g, inp["X"], inp["Wk"], inp["Wq"], inp["Wv"], inp["Watt"], inp["Wmsg"], inp["mu"], heads)
        if tail:
            c["h"] = h
            return hgt_tail_forward(g, h, inp["X"], inp["A"]), c
        return h, c
    raise ValueError(model)


def backward(model: str, g: HeteroGraph, inp: Dict[str, np.ndarray], G: np.ndarray, *, norm=None,
             norm_kind: str = "mean", self_loop: bool = True, slope: float = 0.2,
             heads: int = 1, tail: bool = False) -> Dict[str, np.ndarray]:
    if model == "rgcn":
        if norm is None:
            norm = rgcn_edge_norm(g, norm_kind)
        return rgcn_backward(g, inp["X"], inp["W"], inp["W0"], norm, G, self_loop)
    if model == "rgat":
        return rgat_backward(g, inp["X"], inp["W"], inp["a"], inp["b"], G, slope)
    if model == "hgt":
        args = (g, inp["X"], inp["Wk"], inp["Wq"], inp["Wv"], inp["Watt"], inp["Wmsg"], inp["mu"])
        if not tail:
            return hgt_backward(*args, G, heads)
        h, _ = hgt_forward(*args, heads)
        dh, dA = hgt_tail_backward(g, h, inp["X"], inp["A"], G)
        out = hgt_backward(*args, dh, heads)
        out["dX"] = out["dX"] + G
        out["dA"] = dA
        return out
    raise ValueError(model)
