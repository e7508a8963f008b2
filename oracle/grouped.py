"""ctypes binding of oracle/grouped.c: the fp64 "grouped" oracle (one product per distinct (relation,
node) pair, exact by P:775 §3.3.2), plain C + OpenMP, used to time the oracle on full-size graphs
(bench.py cpu_baseline / --impl reference) and cross-checked against the per-edge
oracle (oracle/layers.py) by tests/test_oracle_grouped.py.

TEST INFRASTRUCTURE (see oracle/__init__.py).  `build()` compiles oracle/libgrouped.so with gcc.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Dict, Optional, Tuple

import numpy as np

from synth.graphs import HeteroGraph

_DIR = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_DIR, "grouped.c")
_LIB = os.path.join(_DIR, "libgrouped.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.run(["gcc", "-O3", "-fopenmp", "-shared", "-fPIC", "-o", _LIB, _SRC, "-lm"],
                       check=True)
    return _LIB


class _Graph(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("e", ctypes.c_int64), ("R", ctypes.c_int32), ("T", ctypes.c_int32),
                ("ntp", ctypes.c_void_p), ("src", ctypes.c_void_p), ("dst", ctypes.c_void_p), ("rel", ctypes.c_void_p)]


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.og_max_threads.restype = ctypes.c_int
        _lib.og_set_threads.argtypes = [ctypes.c_int]
    return _lib


def set_threads(n: int) -> None:
    lib().og_set_threads(int(n))


def max_threads() -> int:
    return int(lib().og_max_threads())


def _p(a: Optional[np.ndarray]):
    return ctypes.c_void_p(0 if a is None else a.ctypes.data)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def forward_backward(model: str, g: HeteroGraph, inp: Dict[str, np.ndarray], G: Optional[np.ndarray] = None, *,
                     norm: Optional[np.ndarray] = None, self_loop: bool = True, slope: float = 0.2
                     ) -> Tuple[np.ndarray, Dict[str, np.ndarray]]:
    """out and (when G is given) the gradients, named as oracle/layers.py names them.  RGCN needs the
    per-edge norm (oracle.layers.rgcn_edge_norm); HGT is the one-head layer without the F2 tail."""
    L = lib()
    keep = []
    ntp = np.ascontiguousarray(g.node_type_ptr, dtype=np.int64)
    src = np.ascontiguousarray(g.src, dtype=np.int32)
    dst = np.ascontiguousarray(g.dst, dtype=np.int32)
    rel = np.ascontiguousarray(g.rel, dtype=np.int32)
    keep += [ntp, src, dst, rel]
    gr = _Graph(g.num_nodes, g.num_edges, g.num_rels, g.num_node_types, ntp.ctypes.data, src.ctypes.data,
                dst.ctypes.data, rel.ctypes.data)
    n, R, T = g.num_nodes, g.num_rels, g.num_node_types
    X = _f64(inp["X"])
    din = X.shape[1]
    Gd = None if G is None else _f64(G)
    grads: Dict[str, np.ndarray] = {}
    if model == "rgcn":
        W, W0 = _f64(inp["W"]), _f64(inp["W0"])
        dout = W.shape[2]
        nrm = _f64(norm)
        out = np.empty((n, dout))
        if Gd is not None:
            grads = {"dX": np.empty((n, din)), "dW": np.empty((R, din, dout))}
            if self_loop:
                grads["dW0"] = np.empty((din, dout))
        rc = L.og_rgcn(ctypes.byref(gr), din, dout, _p(X), _p(W), _p(W0), _p(nrm), int(self_loop), _p(Gd), _p(out),
                       _p(grads.get("dX")), _p(grads.get("dW")), _p(grads.get("dW0")))
    elif model == "rgat":
        W, a, b = _f64(inp["W"]), _f64(inp["a"]), _f64(inp["b"])
        out = np.empty((n, din))
        if Gd is not None:
            grads = {"dX": np.empty((n, din)), "dW": np.empty((R, din, din)), "da": np.empty((R, din)),
                     "db": np.empty((R, din))}
        L.og_rgat.argtypes = [ctypes.c_void_p, ctypes.c_int] + [ctypes.c_void_p] * 4 + [ctypes.c_double] + \
            [ctypes.c_void_p] * 6
        rc = L.og_rgat(ctypes.byref(gr), din, _p(X), _p(W), _p(a), _p(b), float(slope), _p(Gd), _p(out),
                       _p(grads.get("dX")), _p(grads.get("dW")), _p(grads.get("da")), _p(grads.get("db")))
    elif model == "hgt":
        Wk, Wq, Wv, Watt, Wmsg, mu = (_f64(inp[k]) for k in ("Wk", "Wq", "Wv", "Watt", "Wmsg", "mu"))
        d = Watt.shape[2]
        out = np.empty((n, d))
        if Gd is not None:
            grads = {"dX": np.empty((n, din)), "dWk": np.empty((T, din, d)), "dWq": np.empty((T, din, d)),
                     "dWv": np.empty((T, din, d)), "dWatt": np.empty((R, d, d)), "dWmsg": np.empty((R, d, d))}
        rc = L.og_hgt(ctypes.byref(gr), din, d, _p(X), _p(Wk), _p(Wq), _p(Wv), _p(Watt), _p(Wmsg), _p(mu), _p(Gd),
                      _p(out), _p(grads.get("dX")), _p(grads.get("dWk")), _p(grads.get("dWq")),
                      _p(grads.get("dWv")), _p(grads.get("dWatt")), _p(grads.get("dWmsg")))
    else:
        raise ValueError(model)
    if rc != 0:
        raise ValueError("grouped oracle: bad argument")
    return out, grads
