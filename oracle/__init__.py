"""fp64 CPU oracle for one relational-GNN layer (Hector hot path, arxiv 2412.04747 Ch. 3).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import or execute
anything in this package.  The product path (`paper_2412_04747_b200`) never
imports it, and this package never imports the product path; the two share
only the seeded input generators in `synth/`.

Contents
  graph.py   C1 graph-build reference (type sort, dst-CSR, src-CSC, compact pairs)
  layers.py  C3-C5 plain per-edge (vanilla) definitions of RGCN / RGAT / HGT,
             forward and exact backward, in float64
  dense.py   independent dense (matrix-level) formulations used as pins:
             GCN A*XW, g-SpMM / g-SDDMM with a dense masked
             adjacency, GAT / masked dot-product attention
  gemm.py    A1 typed segment GEMM Y[S] = X[G] x W[T] (GEMM template)
  fd.py      central finite differences of L = sum(out * G) (reading g12)
  train.py   F4 training step: stacked layers with ReLU, NLL loss vs random labels
             (P:1062), exact backward through the stack, SGD update
  sample.py  subgraph extraction so that sampled output rows of a large
             graph can be evaluated exactly by the same functions

Readings where the paper is silent are SURVEY.md §8(c) C2 g1-g17, restated in
DESIGN.md "Readings".  Parity status: every function here is pinned by a
`-m "not gpu"` test (tests/test_oracle_*.py); none is "parity unpinned".
"""
