"""Dense matrix-level formulations used to PIN oracle/layers.py (tiny graphs only).

TEST INFRASTRUCTURE (see oracle/__init__.py).  These evaluate the same layers
through a different route than the per-edge loops in layers.py: dense masked
adjacency matrices per relation, transform-then-aggregate at the matrix level,
exactly the g-SpMM / g-SDDMM formulation of P:570-588 §3.2.1, and the textbook
special cases GCN, GAT (one relation) and masked scaled
dot-product attention (HGT with one relation and one node type).
Duplicate (src, dst, rel) triples are not representable densely; callers use
graphs without them (generator default, reading g11).
"""
from __future__ import annotations

import numpy as np

from synth.graphs import HeteroGraph


def adjacency(g: HeteroGraph, r: int, weights=None) -> np.ndarray:
    """A_r[i, j] = weight of edge j -> i with relation r (dense, N x N)."""
    n = g.num_nodes
    A = np.zeros((n, n))
    m = g.rel == r
    w = np.ones(m.sum()) if weights is None else weights[m]
    A[g.dst[m], g.src[m]] = w
    return A


def gcn_dense(g: HeteroGraph, X: np.ndarray, W: np.ndarray) -> np.ndarray:
    """GCN layer A* X W with A*_{ij} = 1/(sqrt(d_out,j) sqrt(d_in,i)) for an edge j -> i."""
    n = g.num_nodes
    A = np.zeros((n, n))
    A[g.dst, g.src] = 1.0
    d_in = A.sum(axis=1)
    d_out = A.sum(axis=0)
    with np.errstate(divide="ignore"):
        ri = np.where(d_in > 0, 1.0 / np.sqrt(d_in), 0.0)
        rj = np.where(d_out > 0, 1.0 / np.sqrt(d_out), 0.0)
    Astar = A * ri[:, None] * rj[None, :]
    return Astar @ X @ W


def gspmm_dense(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    """SpMM C = A x B, c_i = sum_j A_ij b_j, with A given densely."""
    return A @ B


def gsddmm_dense(g: HeteroGraph, A: np.ndarray, B: np.ndarray) -> np.ndarray:
    """SDDMM entries C_ij = a_i . b_j on the edges: returns one value per edge
    e = (j -> i) as A[dst] . B[src] taken from the dense product A B^T."""
    full = A @ B.T
    return full[g.dst, g.src]


def rgcn_dense(g: HeteroGraph, X, W, W0, norm, self_loop=True) -> np.ndarray:
    """Eq. 3.1 as aggregate-then-transform: X W0 + sum_r (C_r o A_r) X W_r."""
    out = X @ W0 if self_loop else np.zeros((g.num_nodes, W.shape[2]))
    for r in range(g.num_rels):
        out = out + (adjacency(g, r, norm) @ X) @ W[r]
    return out


def _masked_softmax_rows(L: np.ndarray, mask: np.ndarray) -> np.ndarray:
    """Row softmax over the masked entries of L (each row: one destination, all its in-edges)."""
    Lm = np.where(mask, L, -np.inf)
    mx = Lm.max(axis=1, keepdims=True)
    mx = np.where(np.isfinite(mx), mx, 0.0)
    ex = np.where(mask, np.exp(Lm - mx), 0.0)
    s = ex.sum(axis=1, keepdims=True)
    return np.divide(ex, s, out=np.zeros_like(ex), where=s > 0)


def rgat_dense(g: HeteroGraph, X, W, a, b, slope=0.2):
    """Multi-relation GAT in matrix form: per relation H_r = X W_r,
    L_r[i, j] = LeakyReLU(H_r[j] . a_r + H_r[i] . b_r) on edges j -> i,
    softmax over the concatenated masked row [L_0 | ... | L_{R-1}] (reading g5),
    out = sum_r alpha_r H_r.  With R = 1 this is the textbook single-head GAT
    e_ij = LeakyReLU(a^T [W h_j || W h_i])."""
    n, R = g.num_nodes, g.num_rels
    Hs = [X @ W[r] for r in range(R)]
    Ls, Ms = [], []
    for r in range(R):
        s = Hs[r] @ a[r]
        t = Hs[r] @ b[r]
        z = t[:, None] + s[None, :]
        Ls.append(np.where(z > 0, z, slope * z))
        Ms.append(adjacency(g, r) > 0)
    Lcat = np.concatenate(Ls, axis=1)
    Mcat = np.concatenate(Ms, axis=1)
    alpha = _masked_softmax_rows(Lcat, Mcat)
    Hcat = np.concatenate(Hs, axis=0)
    return alpha @ Hcat, alpha


def hgt_dense(g: HeteroGraph, X, Wk, Wq, Wv, Watt, Wmsg, mu):
    """Multi-relation masked scaled dot-product attention:
    K_n = X_n Wk_tau(n), Q_n = X_n Wq_tau(n), V_n = X_n Wv_tau(n) (node-typed),
    L_r = mu_r (Q (K Watt_r)^T) / sqrt(d), softmax over the concatenated masked row,
    out = sum_r alpha_r (V Wmsg_r).  One relation and one node type: the textbook
    masked attention softmax(Q K'^T / sqrt(d)) V' restricted to the adjacency."""
    n, R = g.num_nodes, g.num_rels
    tau = g.node_type_of()
    d = Watt.shape[2]
    K = np.stack([X[i] @ Wk[tau[i]] for i in range(n)]) if n else np.zeros((0, d))
    Q = np.stack([X[i] @ Wq[tau[i]] for i in range(n)]) if n else np.zeros((0, d))
    V = np.stack([X[i] @ Wv[tau[i]] for i in range(n)]) if n else np.zeros((0, d))
    Ls, Ms, Vs = [], [], []
    for r in range(R):
        Ls.append(mu[r] * (Q @ (K @ Watt[r]).T) / np.sqrt(d))
        Ms.append(adjacency(g, r) > 0)
        Vs.append(V @ Wmsg[r])
    alpha = _masked_softmax_rows(np.concatenate(Ls, axis=1), np.concatenate(Ms, axis=1))
    return alpha @ np.concatenate(Vs, axis=0), alpha


def edge_alpha_from_dense(g: HeteroGraph, alpha_cat: np.ndarray) -> np.ndarray:
    """Per-edge attention from the concatenated dense alpha (column r*N + src)."""
    n = g.num_nodes
    return alpha_cat[g.dst, g.rel.astype(np.int64) * n + g.src]
