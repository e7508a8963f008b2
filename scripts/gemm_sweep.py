#!/usr/bin/env python
"""D3 d-sweep: the A1 typed segment GEMM Y[S] = X[G] x W[T] on the
mag-shaped compact pair set (segments = relations, G = pair_src), d_in = d_out = d, bf16 on the
tcgen05 path, through the C-ABI (rgnn_segment_gemm).  One JSON line per d: kernel time (CUDA
events via the library's profiler, launch stream), TFLOP/s vs the measured bf16 peak, and
algorithmic GB/s vs the measured HBM peak.  At d = 64 the GEMM is HBM-bound (32 flop/B); the
ridge (~208 flop/B) is crossed near d = 416.

    python scripts/gemm_sweep.py [--dims 64,128,256,512,1024] [--reps 10]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from synth import config_graph  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", default="64,128,256,512,1024")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--no-gather", action="store_true")
    args = ap.parse_args()
    from paper_2412_04747_b200 import Graph, SegmentPlan, rgnn, segment_gemm
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    g = config_graph("mag", seed=1)
    G = Graph.from_hetero(g)
    seg_ptr = G.export("pair_rel_ptr").cpu().tolist()
    pair_src = G.export("pair_src")
    U = int(seg_ptr[-1])
    plan = SegmentPlan(seg_ptr)
    gen = torch.Generator(device="cuda").manual_seed(2)
    for d in [int(x) for x in args.dims.split(",")]:
        # gathered: X has one row per node; ungathered: one row per pair (row r of Y reads row r of X)
        X = (torch.rand(g.num_nodes if not args.no_gather else U, d, device="cuda", generator=gen) * 2 - 1).to(torch.bfloat16)
        W = ((torch.rand(g.num_rels, d, d, device="cuda", generator=gen) * 2 - 1) * (3.0 / d) ** 0.5).to(torch.bfloat16)
        Y = torch.empty(U, d, dtype=torch.bfloat16, device="cuda")
        gather = None if args.no_gather else pair_src
        scratch = torch.empty(g.num_rels * d * d * 2, dtype=torch.uint8, device="cuda")
        for _ in range(3):
            segment_gemm(plan, X, W, gather=gather, out=Y, scratch=scratch)
        torch.cuda.synchronize()
        rgnn.profile_enable(True)
        rgnn.profile_reset()
        for _ in range(args.reps):
            segment_gemm(plan, X, W, gather=gather, out=Y, scratch=scratch)
        torch.cuda.synchronize()
        prof = rgnn.profile_read()
        rgnn.profile_enable(False)
        ms = prof["segment_gemm"]["ms"] / prof["segment_gemm"]["launches"]
        flops = 2.0 * U * d * d
        byts = U * (4 + 2 * d + 2 * d) + g.num_rels * d * d * 2
        tf = flops / ms / 1e9
        gbs = byts / ms / 1e6
        print(json.dumps({"d": d, "rows": U, "segments": g.num_rels, "gather": not args.no_gather,
                          "kernel_ms": round(ms, 4), "tflops": round(tf, 1),
                          "frac_bf16_peak": round(tf / peaks["bf16_tflops"], 3),
                          "frac_bf16_sustained": round(tf / peaks["bf16_tflops_sustained"], 3),
                          "flop_per_byte": round(flops / byts, 1), "gbs": round(gbs, 1),
                          "frac_hbm": round(gbs / peaks["hbm_gbs"], 3),
                          "prep_b_ms": round(prof.get("gemm_tc_prep_b", {}).get("ms", 0) / args.reps, 4)}),
              flush=True)
        del X, W, Y, scratch
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
