"""B200-native relational-GNN layer (RGCN / RGAT / HGT) — the Hector hot path of arxiv 2412.04747.

The compute lives in librgnn.so (csrc/, C-ABI in include/rgnn.h); `rgnn` is its
ctypes binding.  Build with `python -m paper_2412_04747_b200.build`.
"""
from . import rgnn
from .rgnn import Graph, Layer, NllLoss, RGNNError, SegmentPlan, lib, segment_gemm, version
from .train import Stack

__all__ = ["rgnn", "Graph", "Layer", "NllLoss", "RGNNError", "SegmentPlan", "Stack", "lib", "segment_gemm",
           "version"]
