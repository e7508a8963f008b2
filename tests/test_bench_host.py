"""Host-side logic of bench.py (no GPU): the algorithmic-byte model of DESIGN.md §6 and the
training-step accounting.  The formulas are the method's own data movement, so they are checked
against hand-counted cases and structural identities rather than against measurements."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_hgt_bytes_hand_counted():
    # one edge, one pair, one node, d = 8, bf16
    b = bench.algorithmic_bytes("hgt", "bf16", N=1, E=1, U=1, UD=0, R=1, T=1, d_in=8, d=8)
    # forward traversal: per edge the pair index + the [K~|M] row; per node the stats (8 B), the
    # q row (bf16) and the fp32 output row, plus 8 B of softmax statistics
    assert b["hgt_fwd_traverse"] == (4 + 2 * 8 * 2) + (8 + 8 * 2 + 4 * 8 + 8)
    # pair GEMM: index + gathered X row + [K~|M] row written
    assert b["gemm_pairs_fwd"] == 4 + 8 * 2 + 2 * 8 * 2
    # fused A8: index + X row + dKM row read + dX row written
    assert b["pair_bwd_fused"] == 4 + 2 * 8 * 2 + 2 * 8 * 2


@pytest.mark.parametrize("model", ["rgcn", "rgat", "hgt"])
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_bytes_scale_linearly(model, dtype):
    """Doubling E, U and N doubles every kernel's bytes (no hidden constants)."""
    a = bench.algorithmic_bytes(model, dtype, N=100, E=1000, U=300, UD=0, R=4, T=2, d_in=64, d=64)
    b = bench.algorithmic_bytes(model, dtype, N=200, E=2000, U=600, UD=0, R=4, T=2, d_in=64, d=64)
    assert set(a) == set(b)
    for k in a:
        assert b[k] == 2 * a[k], k
    # bf16 tables never cost more than fp32 ones
    if dtype == "bf16":
        f = bench.algorithmic_bytes(model, "f32", N=100, E=1000, U=300, UD=0, R=4, T=2, d_in=64, d=64)
        for k in set(a) & set(f):  # (RGCN's bf16 path adds the bf16 copy of G, "from_f32")
            assert a[k] <= f[k], k


def test_fusion_adjustment():
    alg = bench.algorithmic_bytes("hgt", "bf16", N=10, E=100, U=30, UD=0, R=2, T=2, d_in=64, d=64)
    prof_fused = {"gemm_nodes_dx": {}, "pair_bwd_fused": {}}
    adj = bench.adjust_for_fusions(alg, prof_fused, 30, 10, 64, 2)
    assert adj["gemm_nodes_dx"] == alg["gemm_nodes_dx"] + 30 * (4 + 64 * 2) + 10 * 4
    assert bench.adjust_for_fusions(alg, {"gemm_nodes_dx": {}, "seg_reduce_rows": {}}, 30, 10, 64, 2) == alg


def test_train_bytes_layers():
    one = bench.algorithmic_bytes("rgat", "bf16", N=50, E=500, U=200, UD=0, R=3, T=1, d_in=64, d=64)
    two = bench.train_bytes("rgat", "bf16", N=50, E=500, U=200, R=3, T=1, d=64, layers=2, num_params=1000)
    # layer kernels twice, except the dX kernels (layer 1's input is data)
    assert two["rgat_fwd_traverse"] == 2 * one["rgat_fwd_traverse"]
    assert two["gemm_pairs_dx"] == one["gemm_pairs_dx"]
    # bf16: layer 2 computes dW in the fused A8 kernel, so the separate weight gradient runs once (layer 1)
    assert two["wgrad_pairs"] == one["wgrad_pairs"] and two["pair_bwd_fused"] == one["pair_bwd_fused"]
    assert two["nll_loss"] == 50 * 64 * 8 + 50 * 4
    assert two["relu_fwd"] == 50 * 64 * (4 + 2)
    assert two["sgd_update"] == 1000 * (12 + 2)


def test_single_edge_adjustment():
    a = bench.algorithmic_bytes("hgt", "bf16", N=100, E=1000, U=700, UD=0, R=3, T=1, d_in=64, d=64)
    # below the 30 % threshold nothing moves
    assert bench.adjust_for_single(a, "hgt", 1000, 700, 100, 64, 2) == a
    b = bench.adjust_for_single(a, "hgt", 1000, 700, 500, 64, 2)
    assert b["hgt_bwd_pair"] < a["hgt_bwd_pair"] and b["hgt_bwd_dst"] > a["hgt_bwd_dst"]
    # the pair pass keeps exactly the bytes of the multi-edge pairs
    rest = bench.algorithmic_bytes("hgt", "bf16", N=100, E=500, U=200, UD=0, R=3, T=1, d_in=64, d=64)
    assert b["hgt_bwd_pair"] == rest["hgt_bwd_pair"]
    assert bench.adjust_for_single(a, "rgcn", 1000, 700, 500, 64, 2) == a


def test_single_edge_pairs_count():
    from synth import g7
    g = g7()
    # G7 pairs (rel, src): edges per pair [2, 2, 1, 1, 1] (tests/golden/g7_build.json edge_pair)
    assert bench.single_edge_pairs(g) == 3


def test_d4_terms():
    """SURVEY.md §8(d) D4 evaluated by hand: mag HGT bf16 A7 term E (12 + 4d + db) = 8.36 GB, and the
    per-edge dominant terms 28 + 5db + 4d (HGT), 40 + 2db + 4d (RGAT), 16 + db + 4d (RGCN)."""
    E, N, U, d = 21_111_007, 1_939_743, 3_186_438, 64
    h = bench.d4_bytes("hgt", "bf16", N, E, U, d)
    assert h["rows"]["hgt_bwd_pair"] == E * 396
    assert abs(h["rows"]["hgt_bwd_pair"] / 1e9 - 8.36) < 0.01
    for model, per_edge in (("hgt", 28 + 5 * 128 + 256), ("rgat", 40 + 2 * 128 + 256), ("rgcn", 16 + 128 + 256)):
        a = bench.d4_bytes(model, "bf16", N=0, E=1, U=0, d=64)
        assert a["fwd"] + a["bwd"] == per_edge, model


def test_roofline_counts_only_launched_labels():
    alg = {"a": 1000, "b": 3000, "never": 5000}
    prof = {"a": {"launches": 2, "ms": 2.0}, "b": {"launches": 2, "ms": 4.0}}
    peaks = {"hbm_gbs": 1.0, "source": "t"}
    r = bench.roofline_block(alg, prof, 2, 3.0, peaks, "hgt", "bf16", 1, 1, 1, 64, 1.0, 2.0, False)
    assert r["step_algorithmic_gb"] == 4000 / 1e9
    assert r["kernel"] == "b" and r["ms_per_step"] == 2.0


def test_parse_ncu_dram():
    csv = "\n".join([
        '==PROF== Connected to process',
        '"ID","Process ID","Process Name","Host Name","Kernel Name","Context","Stream","Block Size","Grid Size",'
        '"Device","CC","Section Name","Metric Name","Metric Unit","Metric Value"',
        '"0","1","p","h","void k_hgt_bwd_pair_s<1>(int)","1","7","(256,1,1)","(1,1,1)","0","10.0","","dram__bytes_read.sum","Mbyte","1,000.5"',
        '"0","1","p","h","void k_hgt_bwd_pair_s<1>(int)","1","7","(256,1,1)","(1,1,1)","0","10.0","","dram__bytes_write.sum","Kbyte","500"',
        '"1","1","p","h","void k_hgt_bwd_pair_k<1>(int)","1","7","(256,1,1)","(1,1,1)","0","10.0","","dram__bytes_read.sum","Gbyte","1"',
        '"2","1","p","h","void k_other(int)","1","7","(256,1,1)","(1,1,1)","0","10.0","","dram__bytes_read.sum","Gbyte","9"',
    ])
    tot, n = bench.parse_ncu_dram(csv, "k_hgt_bwd_pair")
    assert n == 2 and abs(tot - (1000.5e6 + 500e3 + 1e9)) < 1


def test_rgat_spmm_bytes_hand_counted():
    # one edge, one pair, one (rel, dst) run, one node, d = 8, bf16: the weighted-SpMM design (default)
    b = bench.algorithmic_bytes("rgat", "bf16", N=1, E=1, U=1, UD=1, R=1, T=1, d_in=8, d=8)
    # A6: pair + rel index, P row, s_p, (alpha, dz) written; node: X row, G + out fp32, stats, G record, dX
    assert b["rgat_bwd_dst"] == (4 + 4 + 16 + 4 + 8) + (16 + 32 + 32 + 8 + 16 + 32)
    # A7 SpMM: CSC dst, CSR position, (alpha, dz), G row; pair: item, dP row, wsum
    assert b["rgat_bwd_pair"] == (4 + 4 + 8 + 16) + (16 + 16 + 4)
    assert b["dpair_sum"] == 8 + 12
    # the recompute design moves the [G | X] record and its 16-byte (lse, G.out) per edge instead
    r = bench.algorithmic_bytes("rgat", "bf16", N=1, E=1, U=1, UD=1, R=1, T=1, d_in=8, d=8, rgat_spmm=False)
    assert r["rgat_bwd_pair"] > b["rgat_bwd_pair"] and "dpair_sum" not in r


def test_single_in_dst_mirror():
    """bench.single_in_dst mirrors layer.cu: RGNN_SINGLE forces; RGAT's SpMM design leaves single-edge
    pairs to the pair pass; otherwise the 30 % threshold."""
    assert bench.single_in_dst("hgt", 1000, 700, 300, env={})
    assert not bench.single_in_dst("hgt", 1000, 700, 100, env={})
    assert not bench.single_in_dst("rgat", 1000, 700, 600, rgat_spmm=True, env={})
    assert bench.single_in_dst("rgat", 1000, 700, 600, rgat_spmm=False, env={})
    assert bench.single_in_dst("rgat", 1000, 700, 0, rgat_spmm=True, env={"RGNN_SINGLE": "1"})
    assert not bench.single_in_dst("rgcn", 1000, 700, 600, env={"RGNN_SINGLE": "1"})
