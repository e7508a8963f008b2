"""Thin ctypes binding over librgnn.so (include/rgnn.h).

Argument marshalling only: every step of the layer runs in the library's CUDA
kernels.  PyTorch supplies device memory (the allocator callbacks and the
workspace tensors), the stream, and the dtype bookkeeping.  There is no CPU
fallback: importing works without a GPU, but every call needs the built
library and a CUDA device, and fails loudly otherwise.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from typing import Dict, Optional

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "librgnn.so")

RGCN, RGAT, HGT = 0, 1, 2
MODELS = {"rgcn": RGCN, "rgat": RGAT, "hgt": HGT}
F32, BF16 = 0, 1
DTYPES = {"f32": F32, "bf16": BF16}
NORMS = {"mean": 0, "sym": 1, "none": 2, "custom": 3}
ARRAYS = ["etype_ptr", "row_ptr", "csr_src", "csr_rel", "csr_eid", "col_ptr", "csc_dst", "csc_rel", "csc_eid",
          "pair_rel_ptr", "pair_src", "edge_pair", "csr_pair", "csc_pair"]
EXPORTED = ["rgnn_last_error", "rgnn_version", "rgnn_graph_build", "rgnn_graph_build_opts", "rgnn_graph_get_info",
            "rgnn_graph_export",
            "rgnn_graph_array_size", "rgnn_graph_destroy", "rgnn_layer_workspace", "rgnn_layer_forward",
            "rgnn_layer_backward", "rgnn_profile_enable", "rgnn_profile_reset", "rgnn_profile_read",
            "rgnn_launch_count", "rgnn_segment_plan_create", "rgnn_segment_plan_destroy",
            "rgnn_segment_gemm_workspace", "rgnn_segment_gemm", "rgnn_relu_forward", "rgnn_relu_backward",
            "rgnn_nll_loss_workspace", "rgnn_nll_loss", "rgnn_sgd_update", "rgnn_comm_unique_id", "rgnn_comm_create",
            "rgnn_comm_destroy", "rgnn_comm_info", "rgnn_comm_exchange_bytes"]
COMM_ID_BYTES = 128

ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_void_p)


class GraphInfo(C.Structure):
    _fields_ = [("num_nodes", C.c_int64), ("num_edges", C.c_int64), ("num_pairs", C.c_int64),
                ("max_in_degree", C.c_int64), ("max_pair_degree", C.c_int64), ("dst_lo", C.c_int64),
                ("dst_hi", C.c_int64), ("num_node_types", C.c_int32), ("num_rels", C.c_int32),
                ("compaction_ratio", C.c_double), ("device_bytes", C.c_int64)]


class GraphOptsC(C.Structure):
    _fields_ = [("compact", C.c_int32), ("reserved", C.c_int32 * 7)]


class LayerDescC(C.Structure):
    _fields_ = [("model", C.c_int32), ("dtype", C.c_int32), ("d_in", C.c_int32), ("d_out", C.c_int32),
                ("self_loop", C.c_int32), ("norm_kind", C.c_int32), ("leaky_slope", C.c_float),
                ("gemm_impl", C.c_int32), ("no_reorder", C.c_int32), ("num_heads", C.c_int32),
                ("hgt_tail", C.c_int32)]


WEIGHT_FIELDS = ["W", "W0", "a", "b", "Wk", "Wq", "Wv", "Watt", "Wmsg", "mu", "edge_norm", "A"]
GRAD_FIELDS = ["dW", "dW0", "da", "db", "dWk", "dWq", "dWv", "dWatt", "dWmsg", "dA"]


class WeightsC(C.Structure):
    _fields_ = [(f, C.c_void_p) for f in WEIGHT_FIELDS]


class GradsC(C.Structure):
    _fields_ = [(f, C.c_void_p) for f in GRAD_FIELDS]


class SgdTensorC(C.Structure):
    _fields_ = [("master", C.c_void_p), ("grad", C.c_void_p), ("shadow", C.c_void_p), ("n", C.c_int64)]


class RGNNError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"rgnn status {code}: {msg}")
        self.code = code


_lib = None


def lib() -> C.CDLL:
    """Load librgnn.so (built by paper_2412_04747_b200.build).  Raises if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run `python -m paper_2412_04747_b200.build` "
                               "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        L.rgnn_last_error.restype = C.c_char_p
        L.rgnn_version.restype = C.c_char_p
        L.rgnn_launch_count.restype = C.c_int64
        for name in EXPORTED:
            if name not in ("rgnn_last_error", "rgnn_version", "rgnn_launch_count"):
                getattr(L, name).restype = C.c_int
        L.rgnn_graph_build.argtypes = [C.c_int64, C.c_int32, C.POINTER(C.c_int64), C.c_int32, C.c_int64,
                                       C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, ALLOC_FN, FREE_FN,
                                       C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]
        L.rgnn_graph_build_opts.argtypes = [C.c_int64, C.c_int32, C.POINTER(C.c_int64), C.c_int32, C.c_int64,
                                            C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                                            C.POINTER(GraphOptsC), ALLOC_FN, FREE_FN, C.c_void_p, C.c_void_p,
                                            C.POINTER(C.c_void_p)]
        L.rgnn_graph_get_info.argtypes = [C.c_void_p, C.POINTER(GraphInfo)]
        L.rgnn_graph_export.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_size_t, C.c_void_p]
        L.rgnn_graph_array_size.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_int64)]
        L.rgnn_graph_destroy.argtypes = [C.c_void_p]
        L.rgnn_layer_workspace.argtypes = [C.c_void_p, C.POINTER(LayerDescC), C.POINTER(C.c_size_t),
                                           C.POINTER(C.c_size_t)]
        L.rgnn_layer_forward.argtypes = [C.c_void_p, C.POINTER(LayerDescC), C.c_void_p, C.POINTER(WeightsC),
                                         C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.rgnn_layer_backward.argtypes = [C.c_void_p, C.POINTER(LayerDescC), C.c_void_p, C.POINTER(WeightsC),
                                          C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(GradsC),
                                          C.c_void_p, C.c_void_p, C.c_void_p]
        L.rgnn_comm_unique_id.argtypes = [C.c_void_p]
        L.rgnn_comm_create.argtypes = [C.c_int32, C.c_int32, C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_void_p)]
        L.rgnn_comm_destroy.argtypes = [C.c_void_p]
        L.rgnn_comm_info.argtypes = [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        L.rgnn_comm_exchange_bytes.argtypes = [C.POINTER(LayerDescC), C.c_int64, C.c_int64, C.POINTER(C.c_int64),
                                               C.POINTER(C.c_int64), C.POINTER(C.c_int32)]
        L.rgnn_segment_plan_create.argtypes = [C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int32), ALLOC_FN,
                                               FREE_FN, C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]
        L.rgnn_segment_plan_destroy.argtypes = [C.c_void_p]
        L.rgnn_segment_gemm_workspace.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                                  C.POINTER(C.c_size_t)]
        L.rgnn_segment_gemm.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p,
                                        C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p,
                                        C.c_size_t, C.c_void_p]
        L.rgnn_relu_forward.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]
        L.rgnn_relu_backward.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.rgnn_nll_loss_workspace.argtypes = [C.c_int64, C.c_int32, C.POINTER(C.c_size_t)]
        L.rgnn_nll_loss.argtypes = [C.c_int64, C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_size_t, C.c_void_p]
        L.rgnn_sgd_update.argtypes = [C.c_int32, C.POINTER(SgdTensorC), C.c_float, C.c_int32, C.c_void_p]
        L.rgnn_profile_enable.argtypes = [C.c_int32]
        L.rgnn_profile_read.argtypes = [C.c_char_p, C.c_size_t]
        _lib = L
    return _lib


def _check(st: int) -> None:
    if st != 0:
        raise RGNNError(st, lib().rgnn_last_error().decode())


def _stream(stream: Optional[torch.cuda.Stream] = None) -> C.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _ptr(t: Optional[torch.Tensor], align: int = 4) -> Optional[int]:
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    if t.data_ptr() % align:
        raise ValueError(f"tensor data must be {align}-byte aligned (the kernels use vector loads)")
    return t.data_ptr()


def version() -> str:
    return lib().rgnn_version().decode()


def launch_count() -> int:
    return int(lib().rgnn_launch_count())


class _TorchAllocator:
    """Allocator callbacks backed by torch's caching allocator; keeps tensors alive by pointer."""

    def __init__(self, device: torch.device):
        self.device = device
        self.live: Dict[int, torch.Tensor] = {}

        def _alloc(nbytes, stream, ctx):
            try:
                t = torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=self.device)
            except RuntimeError:
                return None
            self.live[t.data_ptr()] = t
            return t.data_ptr()

        def _free(ptr, stream, ctx):
            self.live.pop(int(ptr), None)

        self.alloc_cb = ALLOC_FN(_alloc)
        self.free_cb = FREE_FN(_free)


class Graph:
    """A built typed graph (rgnn_graph_build_opts).  src/dst/rel: int32 tensors (moved to the device).
    compact=False builds vanilla materialization (one projected row per edge) for the C ablation."""

    def __init__(self, num_nodes: int, node_type_ptr, num_rels: int, src: torch.Tensor, dst: torch.Tensor,
                 rel: torch.Tensor, dst_range=None, device="cuda", compact: bool = True):
        self.device = torch.device(device)
        self._alloc = _TorchAllocator(self.device)
        ntp = (C.c_int64 * len(node_type_ptr))(*[int(x) for x in node_type_ptr])
        src = torch.as_tensor(src, dtype=torch.int32).to(self.device).contiguous()
        dst = torch.as_tensor(dst, dtype=torch.int32).to(self.device).contiguous()
        rel = torch.as_tensor(rel, dtype=torch.int32).to(self.device).contiguous()
        lo, hi = (0, int(num_nodes)) if dst_range is None else (int(dst_range[0]), int(dst_range[1]))
        h = C.c_void_p()
        e = int(src.numel())
        opts = GraphOptsC()
        opts.compact = int(bool(compact))
        _check(lib().rgnn_graph_build_opts(int(num_nodes), len(node_type_ptr) - 1, ntp, int(num_rels), e,
                                           src.data_ptr() if e else None, dst.data_ptr() if e else None,
                                           rel.data_ptr() if e else None, lo, hi, C.byref(opts),
                                           self._alloc.alloc_cb, self._alloc.free_cb, None, _stream(), C.byref(h)))
        self.handle = h
        self.node_type_ptr = [int(x) for x in node_type_ptr]
        self.num_input_edges = e

    @classmethod
    def from_hetero(cls, g, dst_range=None, device="cuda", compact: bool = True) -> "Graph":
        """From a synth.HeteroGraph-like object (node_type_ptr, num_rels, src, dst, rel)."""
        return cls(int(g.node_type_ptr[-1]), list(g.node_type_ptr), int(g.num_rels), torch.from_numpy(g.src),
                   torch.from_numpy(g.dst), torch.from_numpy(g.rel), dst_range=dst_range, device=device,
                   compact=compact)

    def info(self) -> Dict[str, float]:
        i = GraphInfo()
        _check(lib().rgnn_graph_get_info(self.handle, C.byref(i)))
        return {f: getattr(i, f) for f, _ in GraphInfo._fields_}

    def export(self, name: str) -> torch.Tensor:
        which = ARRAYS.index(name)
        n = C.c_int64()
        _check(lib().rgnn_graph_array_size(self.handle, which, C.byref(n)))
        out = torch.empty(max(n.value, 1), dtype=torch.int32, device=self.device)
        _check(lib().rgnn_graph_export(self.handle, which, out.data_ptr(), out.numel() * 4, _stream()))
        return out[:n.value]

    def close(self) -> None:
        if getattr(self, "handle", None) is not None and self.handle.value:
            lib().rgnn_graph_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Layer:
    """One RGNN layer bound to a graph: rgnn_layer_forward / rgnn_layer_backward.

    weights: dict with the rgnn_weights fields in the layer dtype (mu / edge_norm float32).
    """

    def __init__(self, graph: Graph, model: str, d_in: int, d_out: int, dtype: str = "f32", self_loop: bool = True,
                 norm: str = "mean", leaky_slope: float = 0.2, gemm_impl: int = 0, reorder: bool = True,
                 heads: int = 1, tail: bool = False):
        self.graph = graph
        self.desc = LayerDescC(MODELS[model], DTYPES[dtype], d_in, d_out, int(self_loop), NORMS[norm],
                               float(leaky_slope), int(gemm_impl), int(not reorder), int(heads), int(tail))
        self.model, self.dtype_name = model, dtype
        self.torch_dtype = torch.float32 if dtype == "f32" else torch.bfloat16
        sb, xb = C.c_size_t(), C.c_size_t()
        _check(lib().rgnn_layer_workspace(graph.handle, C.byref(self.desc), C.byref(sb), C.byref(xb)))
        self.saved = torch.empty(sb.value, dtype=torch.uint8, device=graph.device)
        self.scratch = torch.empty(xb.value, dtype=torch.uint8, device=graph.device)
        self.n = graph.info()["num_nodes"]
        self.d_in, self.d_out = d_in, d_out

    def weight_shapes(self) -> Dict[str, tuple]:
        """Expected shape of every weight the model reads (include/rgnn.h rgnn_weights)."""
        i = self.graph.info()
        R, T, di, do = int(i["num_rels"]), int(i["num_node_types"]), self.d_in, self.d_out
        if self.model == "rgcn":
            sh = {"W": (R, di, do)}
            if self.desc.self_loop:
                sh["W0"] = (di, do)
        elif self.model == "rgat":
            sh = {"W": (R, di, do), "a": (R, do), "b": (R, do)}
        else:
            sh = {"Wk": (T, di, do), "Wq": (T, di, do), "Wv": (T, di, do), "Watt": (R, do, do),
                  "Wmsg": (R, do, do), "mu": (R,)}
            if self.desc.hgt_tail:
                sh["A"] = (T, do, do)
        return sh

    def _weights(self, w: Dict[str, torch.Tensor]) -> WeightsC:
        """Check dtype, shape and 16-byte alignment of every weight before its pointer crosses
        the C-ABI (the library takes raw pointers and cannot see a wrong shape)."""
        wc = WeightsC()
        shapes = self.weight_shapes()
        for f, want_shape in shapes.items():
            if f == "mu" and w.get(f) is None:
                continue  # NULL mu => mu_r = 1
            if w.get(f) is None:
                raise ValueError(f"{self.model} layer needs weight {f} of shape {want_shape}")
        for f in WEIGHT_FIELDS:
            t = w.get(f)
            if t is not None:
                want = torch.float32 if f in ("mu", "edge_norm") else self.torch_dtype
                if t.dtype != want:
                    raise TypeError(f"weight {f} must be {want}, got {t.dtype}")
                if f in shapes and tuple(t.shape) != shapes[f]:
                    raise ValueError(f"weight {f} must have shape {shapes[f]}, got {tuple(t.shape)}")
                if f == "edge_norm" and t.numel() != self.graph.num_input_edges:
                    raise ValueError(f"edge_norm must have one value per input edge ({self.graph.num_input_edges})")
                setattr(wc, f, _ptr(t, align=4 if f in ("mu", "edge_norm") else 16))
        return wc

    def _rows(self, name: str, t: torch.Tensor, width: int, dtype: torch.dtype) -> None:
        if t.dtype != dtype:
            raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
        if tuple(t.shape) != (self.n, width):
            raise ValueError(f"{name} must have shape ({self.n}, {width}), got {tuple(t.shape)}")

    def forward(self, X: torch.Tensor, w: Dict[str, torch.Tensor], out: Optional[torch.Tensor] = None,
                comm: Optional["Comm"] = None) -> torch.Tensor:
        """out = layer(X).  With a communicator (multi-GPU), X is the full [N, d_in] buffer whose own
        rows this rank filled; the library all-gathers the other rows into it (in place) and writes
        the owned output rows."""
        self._rows("X", X, self.d_in, self.torch_dtype)
        if out is None:
            out = torch.empty(self.n, self.d_out, dtype=torch.float32, device=X.device)
        self._rows("out", out, self.d_out, torch.float32)
        self._wc = self._weights(w)
        _check(lib().rgnn_layer_forward(self.graph.handle, C.byref(self.desc), _ptr(X, 16), C.byref(self._wc),
                                        _ptr(out, 16), _ptr(self.saved, 16), _ptr(self.scratch, 16),
                                        comm.handle if comm is not None else None, _stream()))
        return out

    def backward(self, X: torch.Tensor, w: Dict[str, torch.Tensor], out: torch.Tensor, dout: torch.Tensor,
                 need_dX: bool = True, grads: Optional[Dict[str, torch.Tensor]] = None,
                 need: Optional[list] = None, comm: Optional["Comm"] = None) -> Dict[str, torch.Tensor]:
        """Gradients of sum(out * dout).  `need` lists weight-gradient names to compute
        (default: all for the model); missing ones are pruned.  With a communicator the owned
        rows of dX hold the full gradient and every weight gradient is summed over the ranks."""
        self._rows("X", X, self.d_in, self.torch_dtype)
        self._rows("out", out, self.d_out, torch.float32)
        self._rows("dout", dout, self.d_out, torch.float32)
        wc = self._weights(w)
        shapes = {k: tuple(v.shape) for k, v in w.items() if v is not None and k not in ("mu", "edge_norm")}
        default = {"rgcn": ["dW", "dW0"] if self.desc.self_loop else ["dW"], "rgat": ["dW", "da", "db"],
                   "hgt": ["dWk", "dWq", "dWv", "dWatt", "dWmsg"] + (["dA"] if self.desc.hgt_tail else [])}[self.model]
        need = default if need is None else need
        grads = dict(grads or {})
        gc = GradsC()
        for name in need:
            if name not in grads:
                grads[name] = torch.empty(shapes[name[1:]], dtype=torch.float32, device=X.device)
            g = grads[name]
            if g.dtype != torch.float32 or tuple(g.shape) != shapes[name[1:]]:
                raise ValueError(f"gradient {name} must be float32 of shape {shapes[name[1:]]}")
            setattr(gc, name, _ptr(g, 16))
        if need_dX and "dX" not in grads:
            grads["dX"] = torch.empty(self.n, self.d_in, dtype=torch.float32, device=X.device)
        if need_dX:
            self._rows("dX", grads["dX"], self.d_in, torch.float32)
        _check(lib().rgnn_layer_backward(self.graph.handle, C.byref(self.desc), _ptr(X, 16), C.byref(wc),
                                         _ptr(out, 16), _ptr(self.saved, 16), _ptr(dout, 16),
                                         _ptr(grads.get("dX"), 16) if need_dX else None, C.byref(gc),
                                         _ptr(self.scratch, 16), comm.handle if comm is not None else None,
                                         _stream()))
        return grads


def comm_unique_id() -> bytes:
    """A fresh NCCL unique id (rgnn_comm_unique_id) to be shared with the other ranks."""
    buf = C.create_string_buffer(COMM_ID_BYTES)
    _check(lib().rgnn_comm_unique_id(buf))
    return buf.raw


class Comm:
    """Library-owned NCCL communicator of one rank (rgnn_comm_create): the layer's multi-GPU exchange
    (all-gather of X in owner chunks, reduce of dX onto the owners, all-reduce of dW) runs inside
    rgnn_layer_forward / rgnn_layer_backward on the library's own stream.  node_ptr: [world+1] owned
    node rows of every rank.  unique_id: the bytes of comm_unique_id() from one rank (share_unique_id)."""

    def __init__(self, rank: int, world: int, node_ptr, unique_id: bytes):
        if len(unique_id) != COMM_ID_BYTES:
            raise ValueError(f"unique_id must be {COMM_ID_BYTES} bytes")
        ptr = [int(x) for x in node_ptr]
        if len(ptr) != world + 1:
            raise ValueError("node_ptr needs world + 1 entries")
        h = C.c_void_p()
        _check(lib().rgnn_comm_create(int(rank), int(world), C.create_string_buffer(unique_id, COMM_ID_BYTES),
                                      (C.c_int64 * len(ptr))(*ptr), C.byref(h)))
        self.handle = h
        self.rank, self.world, self.node_ptr = int(rank), int(world), ptr

    def close(self) -> None:
        if getattr(self, "handle", None) is not None and self.handle.value:
            lib().rgnn_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def exchange_bytes(model: str, dtype: str, d_in: int, d_out: int, num_nodes: int, num_pairs_global: int,
                   heads: int = 1) -> Dict[str, int]:
    """Per-rank bytes of one forward exchange under variant X (all-gather of X) and variant P
    (all-gather of the projected per-pair rows), and the variant the library runs."""
    desc = LayerDescC(MODELS[model], DTYPES[dtype], d_in, d_out, 1, 0, 0.2, 0, 0, heads, 0)
    bx, bp, v = C.c_int64(), C.c_int64(), C.c_int32()
    _check(lib().rgnn_comm_exchange_bytes(C.byref(desc), int(num_nodes), int(num_pairs_global), C.byref(bx),
                                          C.byref(bp), C.byref(v)))
    return {"bytes_x": bx.value, "bytes_p": bp.value, "variant": "XP"[v.value]}


class SegmentPlan:
    """Row tiles of one segmentation for the A1 segment GEMM (rgnn_segment_plan_create).
    seg_ptr: host sequence of num_segments+1 row offsets; seg_weight: optional weight index per segment."""

    def __init__(self, seg_ptr, seg_weight=None, device="cuda"):
        self.device = torch.device(device)
        self._alloc = _TorchAllocator(self.device)
        ptr = [int(x) for x in seg_ptr]
        self.num_segments = len(ptr) - 1
        self.rows = ptr[-1]
        cp = (C.c_int64 * len(ptr))(*ptr)
        cw = None if seg_weight is None else (C.c_int32 * self.num_segments)(*[int(x) for x in seg_weight])
        h = C.c_void_p()
        _check(lib().rgnn_segment_plan_create(self.num_segments, cp, cw, self._alloc.alloc_cb, self._alloc.free_cb,
                                              None, _stream(), C.byref(h)))
        self.handle = h

    def close(self) -> None:
        if getattr(self, "handle", None) is not None and self.handle.value:
            lib().rgnn_segment_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def segment_gemm(plan: SegmentPlan, X: torch.Tensor, W: torch.Tensor, gather: Optional[torch.Tensor] = None,
                 trans_w: bool = False, out_dtype: Optional[torch.dtype] = None, out: Optional[torch.Tensor] = None,
                 scratch: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Y[i] = X[gather[i]] . W[w(seg(i))] for every row of the plan (rgnn_segment_gemm).
    X: [*, K] float32 or bfloat16; W: [num_weights, K, N] (or [num_weights, N, K] with trans_w)."""
    dt = {torch.float32: F32, torch.bfloat16: BF16}[X.dtype]
    if W.dtype != X.dtype:
        raise TypeError("W must have X's dtype")
    K = X.shape[1]
    nw = W.shape[0]
    N = W.shape[1] if trans_w else W.shape[2]
    ydt = out_dtype or torch.float32
    if out is None:
        out = torch.empty(plan.rows, N, dtype=ydt, device=X.device)
    if scratch is None:
        sb = C.c_size_t()
        _check(lib().rgnn_segment_gemm_workspace(plan.handle, dt, K, N, nw, C.byref(sb)))
        scratch = torch.empty(max(sb.value, 1), dtype=torch.uint8, device=X.device)
    if gather is not None and gather.dtype != torch.int32:
        raise TypeError("gather must be int32")
    _check(lib().rgnn_segment_gemm(plan.handle, dt, _ptr(X), _ptr(gather), K, _ptr(W), nw, N, int(trans_w), _ptr(out),
                                   {torch.float32: F32, torch.bfloat16: BF16}[out.dtype], _ptr(scratch),
                                   scratch.numel(), _stream()))
    return out


# ----------------------------------------------------------------- F4 training-step primitives
def relu_forward(h: torch.Tensor, out: Optional[torch.Tensor] = None, dtype: Optional[torch.dtype] = None) -> torch.Tensor:
    """out = max(h, 0) in `dtype` (the next layer's input; rgnn_relu_forward)."""
    if h.dtype != torch.float32:
        raise TypeError("h must be float32")
    if out is None:
        out = torch.empty(h.shape, dtype=dtype or torch.float32, device=h.device)
    _check(lib().rgnn_relu_forward(h.numel(), _ptr(h), _ptr(out), {torch.float32: F32, torch.bfloat16: BF16}[out.dtype],
                                   _stream()))
    return out


def relu_backward(h: torch.Tensor, da: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """dh = da where h > 0 else 0 (rgnn_relu_backward; out may be da)."""
    if out is None:
        out = torch.empty_like(da)
    if not (h.dtype == da.dtype == out.dtype == torch.float32) or h.numel() != da.numel() or da.numel() != out.numel():
        raise TypeError("h, da, out: float32 tensors of one size")
    _check(lib().rgnn_relu_backward(h.numel(), _ptr(h), _ptr(da), _ptr(out), _stream()))
    return out


class NllLoss:
    """Mean NLL of log_softmax rows against int32 labels (rows with label < 0 are unlabelled);
    rgnn_nll_loss.  The loss stays on the device (a float32 scalar tensor)."""

    def __init__(self, n: int, c: int, device="cuda"):
        sb = C.c_size_t()
        _check(lib().rgnn_nll_loss_workspace(int(n), int(c), C.byref(sb)))
        self.n, self.c = int(n), int(c)
        self.scratch = torch.empty(max(sb.value, 1), dtype=torch.uint8, device=device)
        self.loss = torch.empty(1, dtype=torch.float32, device=device)

    def __call__(self, logits: torch.Tensor, labels: torch.Tensor, num_labeled: int,
                 dlogits: Optional[torch.Tensor] = None) -> torch.Tensor:
        if logits.dtype != torch.float32 or tuple(logits.shape) != (self.n, self.c):
            raise TypeError(f"logits must be float32 [{self.n}, {self.c}]")
        if labels.dtype != torch.int32 or labels.numel() != self.n:
            raise TypeError("labels must be int32 [n]")
        _check(lib().rgnn_nll_loss(self.n, self.c, _ptr(logits), _ptr(labels), int(num_labeled), _ptr(self.loss),
                                   _ptr(dlogits), _ptr(self.scratch), self.scratch.numel(), _stream()))
        return self.loss


def sgd_update(tensors, lr: float, shadow_dtype: torch.dtype = torch.float32) -> None:
    """theta -= lr * grad for each (master, grad, shadow-or-None) triple (rgnn_sgd_update, one launch)."""
    arr = (SgdTensorC * max(len(tensors), 1))()
    for i, (m, g, sh) in enumerate(tensors):
        if m.dtype != torch.float32 or g.dtype != torch.float32 or m.numel() != g.numel():
            raise TypeError("master and grad must be float32 of one size")
        if sh is not None and (sh.numel() != m.numel() or sh.dtype != shadow_dtype):
            raise TypeError("shadow must match master's size and shadow_dtype")
        arr[i] = SgdTensorC(_ptr(m), _ptr(g), _ptr(sh), m.numel())
    _check(lib().rgnn_sgd_update(len(tensors), arr, float(lr), {torch.float32: F32, torch.bfloat16: BF16}[shadow_dtype],
                                 _stream()))


def profile_enable(on: bool = True) -> None:
    _check(lib().rgnn_profile_enable(int(on)))


def profile_reset() -> None:
    _check(lib().rgnn_profile_reset())


def profile_read() -> Dict[str, Dict[str, float]]:
    buf = C.create_string_buffer(1 << 16)
    _check(lib().rgnn_profile_read(buf, len(buf)))
    return json.loads(buf.value.decode())
