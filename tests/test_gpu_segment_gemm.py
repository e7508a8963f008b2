"""A1 typed segment GEMM through the C-ABI (rgnn_segment_gemm) vs the fp64 oracle
(oracle/gemm.py, GEMM template P:877): tcgen05 bf16 path at widths 16..1024 (the D3 d-sweep
kernel), ragged tails, empty segments, gathers, shuffled weights, W^T; SIMT f32 path."""
import numpy as np
import pytest
import torch

from oracle import gemm as og
from synth import round_bf16, segment_inputs
from tests.helpers import TOL, rel_err

pytestmark = pytest.mark.gpu


def _run(inp, dtype, out_dtype, trans=False):
    from paper_2412_04747_b200 import SegmentPlan, segment_gemm
    td = torch.bfloat16 if dtype == "bf16" else torch.float32
    X = inp["X"] if dtype == "f32" else round_bf16(inp["X"])
    W = inp["W"] if dtype == "f32" else round_bf16(inp["W"])
    if trans:
        W = np.ascontiguousarray(np.swapaxes(W, 1, 2))
    plan = SegmentPlan(inp["seg_ptr"], inp["seg_weight"])
    Xd = torch.tensor(X, dtype=torch.float32, device="cuda").to(td)
    Wd = torch.tensor(W, dtype=torch.float32, device="cuda").to(td)
    G = None if inp["gather"] is None else torch.tensor(inp["gather"], device="cuda")
    Y = segment_gemm(plan, Xd, Wd, gather=G, trans_w=trans, out_dtype=out_dtype)
    torch.cuda.synchronize()
    ref = og.segment_gemm(X, W, inp["seg_ptr"], inp["gather"], inp["seg_weight"], trans_w=trans)
    return Y.float().cpu().numpy(), ref


# (K, N): the layer widths and the d-sweep widths (N > 256 runs as 256-column blocks)
SHAPES = [(64, 16), (64, 32), (64, 64), (128, 128), (64, 256), (128, 256), (256, 256), (512, 512), (1024, 1024),
          (256, 64), (1024, 128)]


@pytest.mark.parametrize("K,N", SHAPES)
@pytest.mark.parametrize("gather", [True, False])
def test_bf16_tc(K, N, gather):
    lens = [300, 0, 129, 1, 128, 517, 0, 77]
    inp = segment_inputs(7 + K + N, lens, K, N, num_src=900 if gather else 0, gather=gather)
    for out_dtype, tol in ((torch.float32, 1e-4), (torch.bfloat16, TOL["bf16"])):
        got, ref = _run(inp, "bf16", out_dtype)
        assert rel_err(got, ref) < tol, (out_dtype, rel_err(got, ref))


@pytest.mark.parametrize("K,N", [(64, 64), (128, 128), (512, 512)])
def test_bf16_transposed_and_shuffled_weights(K, N):
    inp = segment_inputs(3, [200, 31, 0, 260], K, N, num_src=500, num_weights=6, shuffle_weights=True)
    got, ref = _run(inp, "bf16", torch.float32, trans=True)
    assert rel_err(got, ref) < 1e-4


@pytest.mark.parametrize("K,N", [(16, 16), (64, 64), (32, 256), (128, 128)])
def test_f32_simt(K, N):
    inp = segment_inputs(11, [70, 0, 64, 1, 190], K, N, num_src=400)
    got, ref = _run(inp, "f32", torch.float32)
    assert rel_err(got, ref) < TOL["f32"]


def test_empty_plan_and_errors():
    from paper_2412_04747_b200 import RGNNError, SegmentPlan, segment_gemm
    plan = SegmentPlan([0, 0, 0])
    X = torch.zeros(1, 64, dtype=torch.bfloat16, device="cuda")
    W = torch.zeros(2, 64, 64, dtype=torch.bfloat16, device="cuda")
    assert segment_gemm(plan, X, W).shape == (0, 64)
    plan = SegmentPlan([0, 5])
    with pytest.raises(RGNNError, match="multiple of 64"):
        segment_gemm(plan, torch.zeros(5, 48, dtype=torch.bfloat16, device="cuda"),
                     torch.zeros(1, 48, 64, dtype=torch.bfloat16, device="cuda"))
    with pytest.raises(RGNNError, match="N one of"):
        segment_gemm(plan, torch.zeros(5, 64, dtype=torch.bfloat16, device="cuda"),
                     torch.zeros(1, 64, 48, dtype=torch.bfloat16, device="cuda"))
    with pytest.raises(RGNNError, match="num_weights"):
        segment_gemm(SegmentPlan([0, 5], [3]), torch.zeros(5, 64, dtype=torch.bfloat16, device="cuda"),
                     torch.zeros(1, 64, 64, dtype=torch.bfloat16, device="cuda"))
