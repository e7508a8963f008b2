"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds *no* arithmetic of the method (no projection, attention,
softmax or aggregation).  It only draws graphs and tensors from seeded RNGs and
rounds host tensors to bf16, so that `oracle/` and `paper_2412_04747_b200/`
consume byte-identical inputs without importing one another.

The recipe (node-type sizes, relation endpoints, Zipf relation sizes and
degrees, duplicate redraw, Glorot weights) is SURVEY.md §8(d) D1 and is
restated in DESIGN.md "Input recipe".
"""
from .graphs import (HeteroGraph, g7, load_tsv, dump_tsv, synth_heterograph,
                     config_graph, CONFIGS, random_small_graph)
from .inputs import layer_inputs, random_labels, round_bf16, segment_inputs, stack_inputs, upstream_grad

__all__ = ["HeteroGraph", "g7", "load_tsv", "dump_tsv", "synth_heterograph",
           "config_graph", "CONFIGS", "random_small_graph", "layer_inputs",
           "round_bf16", "segment_inputs", "upstream_grad", "random_labels", "stack_inputs"]
