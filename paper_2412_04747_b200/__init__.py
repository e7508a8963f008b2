"""B200-native relational-GNN layer (RGCN / RGAT / HGT) — the Hector hot path of arxiv 2412.04747.

The compute lives in librgnn.so (csrc/, C-ABI in include/rgnn.h); `rgnn` is its
ctypes binding.  Build with `python -m paper_2412_04747_b200.build`.
"""
from . import rgnn
from .rgnn import Graph, Layer, RGNNError, SegmentPlan, lib, segment_gemm, version

__all__ = ["rgnn", "Graph", "Layer", "RGNNError", "SegmentPlan", "lib", "segment_gemm", "version"]
