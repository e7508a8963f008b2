"""Parity of the non-default kernel designs that the library selects by environment switch (read once per
process, so each case runs in a subprocess): the RGAT recompute pair pass (RGNN_RGATW=0), the
register-resident t-path rows (RGNN_STAGE_Y=0, also what graphs with R * d * 4 > 48 KB run) and the
single-edge pairs resolved in the destination pass of the weighted-SpMM design (RGNN_SINGLE=1, with and
without staged y).
Same oracle and tolerances as tests/test_gpu_layers.py.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASE = """
from synth import config_graph
from synth.graphs import synth_heterograph
from tests.test_gpu_layers import run_case
for dtype in ("f32", "bf16"):
    run_case("rgat", config_graph("aifb", seed=1), 64, 64, dtype)
    g = synth_heterograph([300, 2000], [(1, 0), (0, 0), (1, 1)], rel_sizes=[9000, 4000, 3000],
                          a_src=0.3, a_dst=1.3, seed=5, name="hubs")
    run_case("rgat", g, 64, 64, dtype)
print("ok")
"""


@pytest.mark.parametrize("env", [{"RGNN_RGATW": "0"}, {"RGNN_STAGE_Y": "0"}, {"RGNN_RGATW": "0", "RGNN_STAGE_Y": "0"},
                                 {"RGNN_SINGLE": "1"}, {"RGNN_SINGLE": "1", "RGNN_STAGE_Y_SGL": "1"}])
def test_rgat_switches(env):
    r = subprocess.run([sys.executable, "-c", CASE], cwd=ROOT, env={**os.environ, **env}, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), (env, r.stdout[-2000:], r.stderr[-4000:])


CASE_HGT = """
from synth import config_graph
from tests.test_gpu_layers import run_case
for dtype in ("f32", "bf16"):
    run_case("hgt", config_graph("aifb", seed=1), 64, 64, dtype)
    run_case("hgt", config_graph("tiny", seed=1), 64, 64, dtype)
print("ok")
"""


@pytest.mark.parametrize("env", [{"RGNN_SHORT_PAIR": "1"}, {"RGNN_SPLIT": "0"}, {"RGNN_SHORT": "0"}])
def test_hgt_switches(env):
    """The HGT pair pass with its KI = 2 short-item kernel (RGNN_SHORT_PAIR=1), the staged group kernel
    instead of the split-halves one (RGNN_SPLIT=0), and no short-item kernels anywhere (RGNN_SHORT=0)."""
    r = subprocess.run([sys.executable, "-c", CASE_HGT], cwd=ROOT, env={**os.environ, **env}, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), (env, r.stdout[-2000:], r.stderr[-4000:])
