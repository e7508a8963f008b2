#!/usr/bin/env python
"""Benchmark: one RGNN layer, forward + backward, edges/s (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config mag_hgt] [--impl ours|reference]

Default workload (BASELINE.json configs[3], the configuration the metric is quoted
on): HGT layer, hidden 64, on the ogbn-mag-shaped synthetic heterograph (1.94M
nodes, 4 node types, 21.1M edges, 4 relations), bf16 tensor-core path, full
forward + backward (all weight gradients and dX) per step.

A step = rgnn_layer_forward + rgnn_layer_backward over the whole graph (every row
of SURVEY.md §8(a) A1-A8).  For N > 1 (torchrun) the graph is partitioned by
destination range; each step also all-gathers X (NCCL), reduce-scatters dX and
all-reduces dW; time is the max over ranks.

The JSON line carries: value (device-timed, inputs resident in HBM), e2e (public
API with pinned host buffers, H2D of X and dout and D2H of dX and dW inside the
timed region), roofline of the dominant kernel (algorithmic bytes per launch /
CUDA-event launch time, against MEASURED_PEAKS.json), per-kernel times, clocks
sampled with nvidia-smi during the timed region, and the fp64 oracle timed on
the host cores on a bounded sample (cpu_baseline).
`--impl reference` times the oracle (the reference arm of this tier) instead.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import config_graph, layer_inputs, upstream_grad  # noqa: E402
from synth.inputs import round_bf16  # noqa: E402

METRIC = "RGNN layer fwd+bwd edges/sec (RGAT/HGT, mag-shaped); HBM GB/s vs peak"
UNIT = "edges/s"

BENCH_CONFIGS = {
    # name: graph config, layer, d_in, d_out, dtype, BASELINE.json configs index
    "mag_hgt": dict(graph="mag", model="hgt", d=64, dtype="bf16", baseline=3),
    "mag_hgt_f32": dict(graph="mag", model="hgt", d=64, dtype="f32", baseline=3),
    "mag_hgt_h8": dict(graph="mag", model="hgt", d=64, dtype="bf16", baseline=3, heads=8),
    "mag_rgat": dict(graph="mag", model="rgat", d=64, dtype="bf16", baseline=3),
    "am_rgat": dict(graph="am", model="rgat", d=64, dtype="bf16", baseline=2),
    "am_hgt": dict(graph="am", model="hgt", d=64, dtype="bf16", baseline=2),
    "aifb_hgt": dict(graph="aifb", model="hgt", d=64, dtype="bf16", baseline=1),
    "aifb_rgat": dict(graph="aifb", model="rgat", d=64, dtype="bf16", baseline=1),
    "bgs_rgat": dict(graph="bgs", model="rgat", d=64, dtype="bf16", baseline=1),
    "wikikg2_rgcn": dict(graph="wikikg2", model="rgcn", d=64, dtype="bf16", baseline=4),
    "tiny_rgcn": dict(graph="tiny", model="rgcn", d=16, dtype="f32", baseline=0),
    "mutag_rgat": dict(graph="mutag", model="rgat", d=64, dtype="bf16", baseline=1),
    "fb15k_rgcn": dict(graph="fb15k", model="rgcn", d=64, dtype="bf16", baseline=4),
    "biokg_hgt": dict(graph="biokg", model="hgt", d=64, dtype="bf16", baseline=3),
    # F4: a whole 2-layer training step (layer, ReLU, layer, NLL loss vs random labels, backward, SGD)
    "aifb_rgat_train": dict(graph="aifb", model="rgat", d=64, dtype="bf16", baseline=1, layers=2),
    "bgs_rgat_train": dict(graph="bgs", model="rgat", d=64, dtype="bf16", baseline=1, layers=2),
    "am_rgat_train": dict(graph="am", model="rgat", d=64, dtype="bf16", baseline=2, layers=2),
    "mag_hgt_train": dict(graph="mag", model="hgt", d=64, dtype="bf16", baseline=3, layers=2),
}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": float(d["hbm_gbs"]), "bf16_tflops": float(d["bf16_tflops"]),
                "bf16_tflops_sustained": float(d.get("bf16_tflops_sustained", d["bf16_tflops"])),
                "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "source": "fallback (B200_PROFILING.md)"}


# ----------------------------------------------------------------- algorithmic bytes per launch
def algorithmic_bytes(model, dtype, N, E, U, UD, R, T, d_in, d, rgat_spmm=True):
    """Bytes each kernel must move, per launch.
    Each gathered row counts once per use even if L2 serves it; int32 indices; grads fp32.
    rgat_spmm: RGAT's weighted-SpMM backward (the library default, layer.cu rgat_spmm) instead of the
    recompute design (RGNN_RGATW=0)."""
    b = 2 if dtype == "bf16" else 4
    out = {}
    if model == "hgt":
        out["gemm_pairs_fwd"] = U * (4 + d_in * b + 2 * d * b)
        out["gemm_nodes_fwd"] = N * (d_in * b + d * b)
        out["hgt_fwd_traverse"] = E * (4 + 2 * d * b) + N * (8 + d * b + 4 * d + 8)
        # backward tables (dQ, [dK~|dM]) are stored in the layer dtype (b bytes)
        # A6 also writes the node record [G_v | Q_v] (2d*b) + (m, 1/sum, G.out) (16 B) per node
        out["hgt_bwd_dst"] = E * (4 + 2 * d * b) + N * (16 + d * b + 4 * d + 4 * d + 8 + d * b + 2 * d * b + 16)
        # A7 per edge: CSC dst index, the [G|Q] row of the destination, its 16-B record; per pair: KM row, dKM row
        out["hgt_bwd_pair"] = E * (4 + 2 * d * b + 16) + U * (16 + 2 * d * b + 2 * d * b)
        # dX: per-pair rows dXp = dKM F^T (layer dtype), node rows dX = dQ Wq^T (fp32), then the
        # per-source sum of the pair rows added into dX (seg_reduce_rows)
        out["gemm_pairs_dx"] = U * (2 * d * b + d_in * b)
        out["gemm_nodes_dx"] = N * (d * b + 4 * d_in)
        out["seg_reduce_rows"] = U * (4 + d_in * b) + N * (4 + 8 * d_in)
        out["wgrad_pairs"] = U * (4 + d_in * b + 2 * d * b)
        out["wgrad_nodes"] = N * (d_in * b + d * b)
    elif model == "rgat":
        out["gemm_pairs_fwd"] = U * (4 + d_in * b + d * b + 4)
        out["rgat_fwd_traverse"] = E * (4 + 4 + d * b + 4) + N * (16 + d_in * b + 4 * d + 8)
        if rgat_spmm:
            # A6 per edge: pair + relation index, P row, s_p, and the (alpha, dz) record written; per node:
            # X row, G and out (fp32), stats, the G-only node record written, the t-path dX row written
            out["rgat_bwd_dst"] = E * (4 + 4 + d * b + 4 + 8) + N * (d_in * b + 4 * d + 4 * d + 8 + d * b + 4 * d)
            # A7 weighted SpMM per edge: CSC dst, CSR position, (alpha, dz), the destination's G row; per pair:
            # the work item, dP row and wsum written
            out["rgat_bwd_pair"] = E * (4 + 4 + 8 + d * b) + U * (16 + d * b + 4)
            # B_r: dz summed per (rel, dst) run, then a weighted row sum of X[dst] per relation; da: wsum-weighted P
            out["dpair_sum"] = E * 8 + UD * (4 + 4 + 4)
            out["seg_wsum"] = UD * (4 + 4 + d_in * b) + U * (4 + d * b)
        else:
            # A6 also writes the node record [G_v | X_v] (2d*b) + 16 B
            out["rgat_bwd_dst"] = E * (8 + d * b + 4) + N * (16 + d_in * b + 12 * d + 8 + 2 * d * b + 16)
            # A7 per edge: CSC dst, the destination's [G|X] row and 16-B record; per pair: P row, s, dP, wsum, bx
            out["rgat_bwd_pair"] = E * (4 + 2 * d * b + 16) + U * (16 + 4 + d * b + 4 + d * b + 4 + d * b)
            out["seg_wsum"] = U * (d * b) + U * (4 + d * b)
        out["gemm_pairs_dx"] = U * (d * b + d_in * b)
        out["seg_reduce_rows"] = U * (4 + d_in * b) + N * (4 + 8 * d_in)
        out["wgrad_pairs"] = U * (4 + d_in * b + d * b)
    else:
        out["gemm_pairs_fwd"] = U * (4 + d_in * b + d * b)
        out["gemm_selfloop_fwd"] = N * (d_in * b + 4 * d)
        out["rgcn_fwd_traverse"] = E * (4 + 4 + d * b) + N * (16 + 8 * d)
        out["rgcn_bwd_pair"] = E * (4 + 4 + d * b) + U * (16 + d * b)
        out["gemm_pairs_dx"] = U * (d * b + d_in * b)
        out["gemm_selfloop_dx"] = N * (d * b + 4 * d_in)
        out["seg_reduce_rows"] = U * (4 + d_in * b) + N * (4 + 8 * d_in)
        if b == 2:  # the upstream gradient's bf16 copy (gathered per edge and the self-loop A operand)
            out["from_f32"] = N * d * (4 + b)
        out["wgrad_pairs"] = U * (4 + d_in * b + d * b)
        out["wgrad_selfloop"] = N * (d_in * b + d * b)
    # A8 fused (k_pair_bwd_tc): per pair the X[src] gather, the dP row read once, the dX row written
    k2 = 2 * d if model == "hgt" else d
    out["pair_bwd_fused"] = U * (4 + 2 * d_in * b + k2 * b)
    return out


def dst_rel_pairs(g):
    """Number of distinct (rel, dst) pairs (UD: the (rel, dst) runs of the dst-CSR)."""
    return int(np.unique(g.rel.astype(np.int64) * g.num_nodes + g.dst).size)


def rgat_spmm_on(args):
    """Mirror of layer.cu rgat_spmm: the weighted-SpMM RGAT backward unless reordering is off or RGNN_RGATW=0."""
    return not getattr(args, "no_reorder", False) and os.environ.get("RGNN_RGATW") != "0"


def single_edge_pairs(g):
    """Number of (rel, src) pairs with exactly one edge (host count; the library resolves them in
    the destination-major backward pass when they are >= 30 % of the pairs, layer.cu single_in_dst)."""
    key = g.rel.astype(np.int64) * g.num_nodes + g.src
    _, cnt = np.unique(key, return_counts=True)
    return int((cnt == 1).sum())


def single_in_dst(model, E, U, U1, rgat_spmm=True, env=None):
    """Mirror of layer.cu single_in_dst: RGNN_SINGLE forces it; RGAT's weighted-SpMM design leaves the
    single-edge pairs to the pair pass; otherwise on when they are >= 30 % of the pairs."""
    env = os.environ if env is None else env
    if model not in ("hgt", "rgat"):
        return False
    if env.get("RGNN_SINGLE") in ("0", "1"):
        return env["RGNN_SINGLE"] == "1"
    if model == "rgat" and rgat_spmm:
        return False
    return 10 * U1 >= 3 * U


def adjust_for_single(alg, model, E, U, U1, d, b, rgat_spmm=True, env=None):
    """Move the single-edge pairs' bytes from the pair-major label to the destination-major one:
    the pair pass no longer gathers their node records; the dst pass reads a 1-byte flag per edge
    and writes their gradient rows (HGT [dK~ | dM]; RGAT dP, bx, wsum and reads a_r)."""
    if not single_in_dst(model, E, U, U1, rgat_spmm, env):
        return alg
    alg = dict(alg)
    if model == "rgat" and rgat_spmm:  # dst pass writes their dP row + wsum; the pair pass skips them
        alg["rgat_bwd_pair"] -= U1 * (4 + 4 + 8 + d * b) + U1 * (16 + d * b + 4)
        alg["rgat_bwd_dst"] += E * 1 + U1 * (d * b + 4)
        return alg
    if model == "hgt":
        alg["hgt_bwd_pair"] -= U1 * (4 + 2 * d * b + 16) + U1 * (16 + 2 * d * b + 2 * d * b)
        alg["hgt_bwd_dst"] += E * 1 + U1 * (2 * d * b)
    else:
        alg["rgat_bwd_pair"] -= U1 * (4 + 2 * d * b + 16) + U1 * (16 + 4 + d * b + 4 + d * b + 4 + d * b)
        alg["rgat_bwd_dst"] += E * 1 + U1 * (d * b + d * b + d * b + 4)
    return alg


def adjust_for_fusions(alg, prof, U, N, d_in, b):
    """Kernel labels that absorbed another kernel's work carry its bytes: when the per-source
    reduction of the pair dX rows runs in the HGT node GEMM's epilogue (no seg_reduce_rows launch),
    gemm_nodes_dx also gathers the pair rows (U rows + list) and skips dX's write + re-read."""
    if "gemm_nodes_dx" in prof and "seg_reduce_rows" not in prof and "gemm_nodes_dx" in alg:
        alg = dict(alg)
        alg["gemm_nodes_dx"] += U * (4 + d_in * b) + N * 4
    return alg


def d4_bytes(model, dtype, N, E, U, d):
    """what the method itself must move per fwd and bwd (fused design, int32
    indices, fp32 gradients, b = stored feature bytes), plus the D4 term of each traversal row
    (A3-A5 forward, A6 dst-major, A7 pair-major) for the dominant-kernel comparison."""
    b = 2 if dtype == "bf16" else 4
    db = d * b
    if model == "rgcn":
        fwd = U * 2 * db + E * (8 + db) + N * (2 * db + 8 * d + 4)
        bwd = E * (8 + 4 * d) + U * (8 * d + db) + N * (8 * d + db)
        rows = {"rgcn_fwd_traverse": E * (8 + db) + N * (8 * d + 4), "rgcn_bwd_pair": E * (8 + 4 * d)}
    elif model == "rgat":
        fwd = U * (2 * db + 4) + E * (10 + db) + N * (db + 4 * d + 12)
        bwd = E * (18 + db) + E * (12 + 4 * d) + U * (8 * d + db) + N * (8 * d + db + 4)
        rows = {"rgat_fwd_traverse": E * (10 + db) + N * (db + 4 * d + 12), "rgat_bwd_dst": E * (18 + db),
                "rgat_bwd_pair": E * (12 + 4 * d)}
    else:
        fwd = U * 3 * db + N * 3 * db + E * (4 + 2 * db) + N * (4 * d + 12)
        bwd = E * (12 + 2 * db) + E * (12 + 4 * d + db) + U * (12 * d + db) + N * (16 * d + db + 4)
        rows = {"hgt_fwd_traverse": E * (4 + 2 * db) + N * (4 * d + 12), "hgt_bwd_dst": E * (12 + 2 * db),
                "hgt_bwd_pair": E * (12 + 4 * d + db)}
    return {"fwd": fwd, "bwd": bwd, "rows": rows}


# kernel-name regex of each traversal label (every launch of the label: warp, group and short halves)
LABEL_KERNELS = {"hgt_bwd_pair": "k_hgt_bwd_pair", "hgt_bwd_dst": "k_hgt_bwd_dst", "hgt_fwd_traverse": "k_hgt_fwd",
                 "rgat_bwd_pair": "k_rgat_bwd_pair|k_pair_spmm", "rgat_bwd_dst": "k_rgat_bwd_dst",
                 "rgat_fwd_traverse": "k_rgat_fwd", "rgcn_bwd_pair": "k_rgcn_bwd_pair",
                 "rgcn_fwd_traverse": "k_rgcn_fwd", "pair_bwd_fused": "k_pair_bwd_tc|k_pair_bwd_ws"}


def source_hash() -> str:
    """sha1 over the library sources (csrc + include): ties an ncu capture to the build it measured."""
    import glob
    import hashlib
    h = hashlib.sha1()
    files = sorted(glob.glob(os.path.join(ROOT, "paper_2412_04747_b200", "csrc", "*")) +
                   glob.glob(os.path.join(ROOT, "include", "*.h")))
    for f in files:
        h.update(os.path.basename(f).encode())
        h.update(open(f, "rb").read())
    return h.hexdigest()[:12]


def parse_ncu_dram(csv_text: str, pattern: str):
    """Sum dram__bytes_read.sum + dram__bytes_write.sum over the launches whose name contains
    `pattern` in an `ncu --csv` (--page raw or metric list) log; returns (bytes, launches)."""
    import csv
    import io
    lines = [l for l in csv_text.splitlines() if l.startswith('"')]
    if not lines:
        return None, 0
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    h = rows[0]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    if "Metric Name" in h:  # long format: one row per (launch, metric)
        ki, ii, mi, ui, vi = (h.index("Kernel Name"), h.index("ID"), h.index("Metric Name"), h.index("Metric Unit"),
                              h.index("Metric Value"))
        tot, ids = 0.0, set()
        for r in rows[1:]:
            if pattern in r[ki] and r[mi] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                tot += float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
                ids.add(r[ii])
        return (tot if ids else None), len(ids)
    return None, 0


def ncu_traffic_in_run(args, label):
    """DRAM bytes per step of `label`, measured now on this build: ncu (two DRAM counters, cold-cache
    serialised replays) over a child bench run of the same config (3 warm-up + 1 step), bytes
    summed over the label's launches and divided by the 4 steps run.  None when ncu is absent."""
    import shutil
    ncu = shutil.which("ncu") or ("/usr/local/cuda/bin/ncu" if os.path.exists("/usr/local/cuda/bin/ncu") else None)
    pat = LABEL_KERNELS.get(label)
    if ncu is None or pat is None:
        return None
    cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum", "--clock-control", "none", "--csv",
           "-k", f"regex:{pat}", sys.executable, os.path.abspath(__file__), "--config", args.config, "--steps", "1",
           "--warmup", "3", "--no-cpu-baseline", "--no-e2e", "--no-ncu"]
    if args.a_dst is not None:
        cmd += ["--a-dst", str(args.a_dst)]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=args.ncu_timeout)
    except (subprocess.TimeoutExpired, OSError):
        return None
    tot, n = parse_ncu_dram(r.stdout, pat)
    if tot is None:
        return None
    return {"bytes_per_step": tot / 4.0, "launches": n, "steps": 4, "source_hash": source_hash(),
            "how": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:{pat} "
                   f"over bench.py --config {args.config} --steps 1 --warmup 3 (this build, this run)"}


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 50 ms (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.samples = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "50", "-i", str(self.dev)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except (FileNotFoundError, OSError):
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.samples.append((time.time(), parts))

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self, t0, t1):
        def parse(rows):
            mhz, mx, reasons = [], [], set()
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            for _, p in rows:
                try:
                    mhz.append(float(p[1]))
                    mx.append(float(p[2]))
                except ValueError:
                    continue
                for nm, v in zip(names, p[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
            return mhz, mx, reasons
        inside = [s for s in self.samples if t0 <= s[0] <= t1]
        window = "timed region"
        if not inside:  # timed region shorter than the sampling period: nearest samples
            inside = sorted(self.samples, key=lambda s: abs(s[0] - 0.5 * (t0 + t1)))[:3]
            window = "nearest samples (timed region shorter than 50 ms sampling)"
        mhz, mx, reasons = parse(inside)
        if not mhz:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0, "window": "unavailable"}
        return {"sm_mhz": float(np.median(mhz)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(mhz), "window": window}


BAD_REASONS = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
KERNEL_TIMING = {
    False: "per-kernel times (kernels, roofline.achieved) from a second timed pass of the same K steps with CUDA "
           "events around every library launch on its stream; the headline pass carries none (they add ~0.13 ms "
           "to a mag step)",
    True: "per-kernel times from CUDA events around every library launch inside the headline timed region",
}


# ----------------------------------------------------------------- CPU oracle baseline
def cpu_oracle_sample(g, model, inp, Gh, target_s=15.0, seed=0):
    """Time the fp64 oracle (as it stands) on a bounded sample of the workload: the in-edge
    subgraph of random destinations (exact per-destination computation), relabelled."""
    from oracle import layers as L
    from oracle import sample as S
    try:
        from threadpoolctl import threadpool_info
        threads = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        threads = os.cpu_count() or 1
    rng = np.random.default_rng(seed)
    n_dst = max(1, int(2000 * 10.0 / max(1.0, g.num_edges / g.num_nodes)))
    elapsed, edges, last = 0.0, 0, None
    while True:
        dsts = rng.choice(g.num_nodes, size=min(n_dst, g.num_nodes), replace=False)
        _, eids = S.in_edge_subgraph(g, dsts)
        sub, nodes = S.compact_subgraph(g, eids)
        loc = {k: (v[nodes] if k == "X" else v) for k, v in inp.items()}
        kw = {"norm": L.rgcn_edge_norm(g, "mean")[eids]} if model == "rgcn" else {}
        t = time.perf_counter()
        L.forward(model, sub, loc, **kw)
        L.backward(model, sub, loc, Gh[nodes], **kw)
        dt = time.perf_counter() - t
        elapsed += dt
        edges += sub.num_edges
        last = (len(dsts), sub.num_edges)
        if elapsed >= 0.5 * target_s or n_dst >= g.num_nodes:
            break
        n_dst = int(min(g.num_nodes, n_dst * max(2.0, 0.6 * target_s / max(dt, 1e-3))))
    return {"value": edges / elapsed, "unit": UNIT, "cores": int(threads), "kind": "oracle", "cpu_model": cpu_model(),
            "nproc": os.cpu_count(),
            "sample": f"fp64 numpy oracle, vanilla per-edge {model.upper()} fwd+bwd on in-edge subgraphs of random "
                      f"destinations: {edges} edges in {elapsed:.1f} s (last sample {last[0]} dst / {last[1]} edges)",
            "seconds": elapsed}


def cpu_oracle_grouped(g, model, inp, Gh, max_edges=None, threads=None, seed=0):
    """Time the fp64 oracle in its grouped mode (oracle/grouped.c: plain C + OpenMP, one product per
    distinct (relation, node) pair -- exact by P:775 -- cross-checked against the per-edge oracle by
    tests/test_oracle_grouped.py) on the FULL graph, or, with max_edges, on the in-edge subgraph of
    random destinations holding about that many edges."""
    from oracle import grouped as OG
    from oracle import layers as L
    from oracle import sample as S
    threads = int(threads or os.cpu_count() or 1)
    OG.set_threads(threads)
    norm_full = L.rgcn_edge_norm(g, "mean") if model == "rgcn" else None
    if max_edges is None or max_edges >= g.num_edges:
        sub, loc, Gs, norm = g, inp, Gh, norm_full
        what = f"full graph ({g.num_nodes} nodes, {g.num_edges} edges)"
    else:
        rng = np.random.default_rng(seed)
        n_dst = max(1, int(g.num_nodes * max_edges / max(1, g.num_edges)))
        dsts = rng.choice(g.num_nodes, size=min(n_dst, g.num_nodes), replace=False)
        _, eids = S.in_edge_subgraph(g, dsts)
        sub, nodes = S.compact_subgraph(g, eids)
        loc = {k: (v[nodes] if k == "X" else v) for k, v in inp.items()}
        Gs = Gh[nodes]
        norm = None if norm_full is None else norm_full[eids]
        what = f"in-edge subgraph of {len(dsts)} random destinations ({sub.num_edges} edges)"
    kw = {"norm": norm} if model == "rgcn" else {}
    t = time.perf_counter()
    OG.forward_backward(model, sub, loc, Gs, **kw)
    dt = time.perf_counter() - t
    return {"value": sub.num_edges / dt, "unit": UNIT, "cores": threads, "kind": "oracle", "cpu_model": cpu_model(),
            "nproc": os.cpu_count(),
            "sample": f"fp64 grouped oracle (oracle/grouped.c, {threads} OpenMP threads), {model.upper()} fwd+bwd on "
                      f"the {what} in {dt:.1f} s",
            "seconds": dt}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def single_thread(fn, target_s):
    """the oracle timed a second time on one host thread (BLAS limited to 1)."""
    try:
        from threadpoolctl import threadpool_limits
    except Exception:
        return None
    with threadpool_limits(limits=1):
        r = fn(target_s)
    return {"value": r["value"], "unit": r["unit"], "cores": 1, "sample": r["sample"]}


def roofline_block(alg, prof, steps, ms_per_step, peaks, model, dtype, N, E, U, d, t_fwd, t_bwd, infer):
    """Per-kernel view + the dominant label's roofline, three ways: its algorithmic bytes (the
    kernel-level model), the SURVEY.md §8(d) D4 term of its row, and (filled in by the
    caller) ncu DRAM bytes.  Step-level bytes count only the labels that launched in this run."""
    hbm = peaks["hbm_gbs"]
    tot_ms = sum(x["ms"] for x in prof.values())
    kernels = {k: {"launches_per_step": v["launches"] / steps, "ms_per_step": v["ms"] / steps,
                   "share": v["ms"] / max(tot_ms, 1e-9)} for k, v in prof.items()}
    for k in kernels:
        if alg.get(k):
            kernels[k]["algorithmic_bytes_per_step"] = int(alg[k])
            kernels[k]["achieved_gbs"] = alg[k] / (kernels[k]["ms_per_step"] / 1e3) / 1e9
    ran = {k: v for k, v in alg.items() if k in prof}
    d4 = d4_bytes(model, dtype, N, E, U, d)
    d4_step = d4["fwd"] + (0 if infer else d4["bwd"])
    out = {"bound": "hbm", "peak": hbm, "unit": "GB/s", "peak_source": peaks["source"],
           "step_algorithmic_gb": sum(ran.values()) / 1e9,
           "step_achieved_gbs": sum(ran.values()) / (ms_per_step / 1e3) / 1e9,
           "step_frac": sum(ran.values()) / (ms_per_step / 1e3) / 1e9 / hbm,
           "step_d4_gb": d4_step / 1e9, "step_d4_frac": d4_step / (ms_per_step / 1e3) / 1e9 / hbm,
           "d4_fwd_gb": d4["fwd"] / 1e9, "d4_bwd_gb": d4["bwd"] / 1e9,
           "t_fwd_ms": t_fwd, "t_bwd_ms": t_bwd,
           "fwd_d4_frac": d4["fwd"] / (t_fwd / 1e3) / 1e9 / hbm if t_fwd else None,
           "bwd_d4_frac": d4["bwd"] / (t_bwd / 1e3) / 1e9 / hbm if t_bwd else None,
           "kernel": None, "traffic": None, "_kernels": kernels}
    dom = max((k for k in prof if alg.get(k)), key=lambda k: prof[k]["ms"], default=None)
    if dom is None:
        return out
    ms_k = kernels[dom]["ms_per_step"]
    achieved = alg[dom] / (ms_k / 1e3) / 1e9
    out.update({"kernel": dom, "achieved": achieved, "frac": achieved / hbm, "frac_of_8TBps": achieved / 8000.0,
                "algorithmic_bytes_per_step": int(alg[dom]), "launches_per_step": kernels[dom]["launches_per_step"],
                "ms_per_step": ms_k,
                "note": "bytes and time per step of the kernel label (all its launches in one step); frac uses the "
                        "kernel-level byte model, d4_frac the SURVEY.md §8(d) D4 term of the label's row"})
    if dom in d4["rows"]:
        out["d4_bytes_per_step"] = int(d4["rows"][dom])
        out["d4_frac"] = d4["rows"][dom] / (ms_k / 1e3) / 1e9 / hbm
    return out


# ----------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="mag_hgt", choices=sorted(BENCH_CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--gemm-impl", type=int, default=0)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--cuda-graph", action="store_true",
                    help="N=1: capture one fwd+bwd step in a CUDA graph and replay it (launch-bound small graphs); "
                         "per-kernel times then come from a separate un-captured profiling pass")
    ap.add_argument("--no-compact", action="store_true",
                    help="vanilla materialization (one projected row per edge): the C ablation of tab:optimizations")
    ap.add_argument("--no-reorder", action="store_true",
                    help="linear-operator reordering off (HGT): the R ablation of tab:optimizations")
    ap.add_argument("--a-dst", type=float, default=None,
                    help="destination Zipf exponent of the generator (SURVEY.md §8(d) D1 load-balance sensitivity "
                         "points: 0 = uniform in-degrees, 1.2 = heavier skew; default the config's 0.8)")
    ap.add_argument("--profile-in-timed", type=int, default=0,
                    help="0 (default): the headline timed region has no per-launch CUDA events (they cost ~0.13 ms "
                         "per mag step); the per-kernel times come from a second timed pass of the same K steps with "
                         "them.  1: one timed pass with per-launch events (the round-1 behaviour)")
    ap.add_argument("--no-ncu", action="store_true",
                    help="skip the in-run ncu DRAM-traffic capture of the dominant kernel (roofline.traffic)")
    ap.add_argument("--ncu-timeout", type=float, default=300.0)
    ap.add_argument("--comm", action="store_true",
                    help="N=1: run through a world-1 library communicator (the multi-GPU code path on one GPU)")
    ap.add_argument("--infer", action="store_true",
                    help="inference: a step is the forward pass only (the 'Inference' columns of tab:optimizations)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = BENCH_CONFIGS[args.config]

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return run_reference(args, cfg, world, rank)
    if cfg.get("layers", 1) > 1:
        return run_train(args, cfg, world, rank, local_rank)

    import torch
    import torch.distributed as dist
    from paper_2412_04747_b200 import Graph, Layer, rgnn
    from paper_2412_04747_b200 import dist as D

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    g = config_graph(cfg["graph"], seed=1, a_dst=args.a_dst)
    model, d, dtype = cfg["model"], cfg["d"], cfg["dtype"]
    ranges = D.partition_ranges(g.dst, g.num_nodes, world)
    lo, hi = ranges[rank]
    G = Graph.from_hetero(g, dst_range=(lo, hi) if world > 1 else None, device=dev, compact=not args.no_compact)
    info = G.info()
    inp = layer_inputs(model, g, d, d)
    if dtype == "bf16":
        inp = {k: (round_bf16(v) if k not in ("mu",) else v) for k, v in inp.items()}
    Gh = upstream_grad(g.num_nodes, d)
    td = torch.float32 if dtype == "f32" else torch.bfloat16
    w = {k: torch.tensor(np.asarray(v, np.float32), device=dev).to(torch.float32 if k == "mu" else td)
         for k, v in inp.items() if k != "X"}
    # X: a full [N, d] buffer per rank; this rank fills its own rows, the library's forward
    # all-gathers the others into it (NCCL, in place) when N > 1
    X_full = torch.tensor(np.asarray(inp["X"], np.float32), device=dev).to(td)
    if world > 1:
        X_full[:lo] = float("nan")
        X_full[hi:] = float("nan")
    X_own = X_full[lo:hi]
    dout = torch.tensor(Gh, dtype=torch.float32, device=dev)  # the layer reads the owned rows only
    comm = None
    if world > 1:
        comm = D.make_comm(ranges)
    elif args.comm:  # exercise the library-owned exchange path on one GPU (a world-1 NCCL communicator)
        comm = rgnn.Comm(0, 1, D.node_ptr(ranges), rgnn.comm_unique_id())
    layer = Layer(G, model, d, d, dtype=dtype, gemm_impl=args.gemm_impl, reorder=not args.no_reorder,
                  heads=cfg.get("heads", 1))
    wkeys = {"rgcn": ["dW", "dW0"], "rgat": ["dW", "da", "db"], "hgt": ["dWk", "dWq", "dWv", "dWatt", "dWmsg"]}[model]
    grads = {k: torch.empty(w[k[1:]].shape, dtype=torch.float32, device=dev) for k in wkeys}
    grads["dX"] = torch.empty(g.num_nodes, d, dtype=torch.float32, device=dev)
    out = torch.empty(g.num_nodes, d, dtype=torch.float32, device=dev)

    def step(Xb, dout_b=None, mid=None, bufs=None):
        """One layer forward + backward through the public API; with N > 1 the exchange (X
        all-gather, dX reduce onto the owners, dW all-reduce) runs inside the library calls."""
        o, gs = (out, grads) if bufs is None else bufs
        layer.forward(Xb, w, out=o, comm=comm)
        if mid is not None:
            mid()
        if args.infer:
            return o
        gr = layer.backward(Xb, w, o, dout if dout_b is None else dout_b, grads=gs, need=wkeys, comm=comm)
        return gr["dX"]

    for _ in range(args.warmup):
        step(X_full)
    torch.cuda.synchronize()
    graph = None
    if args.cuda_graph and world == 1:
        cs = torch.cuda.Stream()
        cs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cs):
            step(X_full)  # warm the capture stream
        torch.cuda.current_stream().wait_stream(cs)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step(X_full)
        torch.cuda.synchronize()

    sampler = ClockSampler(local_rank)
    sampler.start()
    time.sleep(0.15)

    prof_on = [bool(args.profile_in_timed)]

    def timed(K, use_graph=False):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        rgnn.profile_reset()
        rgnn.profile_enable(not use_graph and prof_on[0])
        n0 = rgnn.launch_count()
        s = torch.cuda.current_stream()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
        evm = [torch.cuda.Event(enable_timing=True) for _ in range(K)]  # after each step's forward
        t0 = time.time()
        ev[0].record(s)
        for i in range(K):
            if use_graph:
                graph.replay()
            else:
                step(X_full, mid=lambda i=i: evm[i].record(s))
            ev[i + 1].record(s)
        torch.cuda.synchronize()
        t1 = time.time()
        if world > 1:
            dist.barrier()
        launches = rgnn.launch_count() - n0
        prof = rgnn.profile_read()
        rgnn.profile_enable(False)
        ms = ev[0].elapsed_time(ev[K])
        per_step[:] = [ev[i].elapsed_time(ev[i + 1]) for i in range(K)]
        if not use_graph:
            fwd_bwd[:] = [(ev[i].elapsed_time(evm[i]), evm[i].elapsed_time(ev[i + 1])) for i in range(K)]
        return ms, launches, prof, t0, t1

    use_graph = graph is not None
    per_step = []  # per-step device times of the last timed() call (D2: median and mean)
    fwd_bwd = []   # per-step (t_fwd, t_bwd) of the last un-captured timed() call (D2)
    ms, launches, prof, t0, t1 = timed(args.steps, use_graph)
    per_step_timed = list(per_step)
    time.sleep(0.12)
    clocks = sampler.summary(t0, t1)
    remeasured = False
    if set(clocks["reasons"]) & BAD_REASONS:
        remeasured = True
        ms, launches, prof, t0, t1 = timed(args.steps, use_graph)
        per_step_timed = list(per_step)
        time.sleep(0.12)
        clocks = sampler.summary(t0, t1)
    fwd_bwd_timed = list(fwd_bwd)
    if use_graph or not args.profile_in_timed:
        # per-kernel attribution: a second timed pass of the same K steps with per-launch CUDA events on each
        # launch's stream (graph replays cannot carry them; in the headline pass they would perturb the step)
        prof_on[0] = True
        _, launches, prof, _, _ = timed(args.steps, False)
        prof_on[0] = bool(args.profile_in_timed)
    sampler.stop()
    if fwd_bwd_timed:  # the headline pass's split (an un-captured pass: the graph path keeps the profiling pass's)
        fwd_bwd[:] = fwd_bwd_timed
    t_fwd = float(np.median([f for f, _ in fwd_bwd])) if fwd_bwd else None
    t_bwd = float(np.median([b_ for _, b_ in fwd_bwd])) if fwd_bwd and not args.infer else None
    if world > 1:
        tms = torch.tensor([ms], device=dev)
        dist.all_reduce(tms, op=dist.ReduceOp.MAX)
        ms = float(tms.item())
    ms_per_step = ms / args.steps
    value = g.num_edges * args.steps / (ms / 1e3)

    # ---- e2e through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        Xh = X_own.cpu().pin_memory()            # the owned rows of X and dout, per step H2D
        douth = dout[lo:hi].cpu().pin_memory()
        dwh = {k: torch.empty(grads[k].shape, dtype=torch.float32).pin_memory() for k in wkeys}
        outh = torch.empty(out.shape, dtype=torch.float32).pin_memory()
        own_rows = slice(lo, hi) if world > 1 else slice(0, g.num_nodes)
        dxh = None if args.infer else torch.empty(hi - lo, d, dtype=torch.float32).pin_memory()
        ds = torch.cuda.Stream(device=dev)  # D2H of the results (second copy engine)
        # results double-buffered too: step i+1 computes into the other buffers while step i's are read
        rbufs = [(out, grads), (torch.empty_like(out), {k: torch.empty_like(v) for k, v in grads.items()})]
        results_ready = [torch.cuda.Event() for _ in range(2)]
        results_read = [torch.cuda.Event() for _ in range(2)]
        # double-buffered: the H2D of step i+1's inputs (copy stream) overlaps step i's kernels
        Xd = [X_full.clone() for _ in range(2)]
        doutd = [dout.clone() for _ in range(2)]
        cs = torch.cuda.Stream(device=dev)
        copied = [torch.cuda.Event() for _ in range(2)]
        consumed = [torch.cuda.Event() for _ in range(2)]
        h2d = Xh.numel() * Xh.element_size() + (0 if args.infer else douth.numel() * douth.element_size())
        d2h = (hi - lo) * d * 4 * (1 if args.infer else 2) + (0 if args.infer else sum(v.numel() * 4 for v in dwh.values()))

        def issue_copy(k):
            with torch.cuda.stream(cs):
                cs.wait_event(consumed[k])  # the step that last read buffer k has finished
                Xd[k][lo:hi].copy_(Xh, non_blocking=True)
                if not args.infer:
                    doutd[k][lo:hi].copy_(douth, non_blocking=True)
                copied[k].record(cs)

        def e2e_run(K):
            s = torch.cuda.current_stream()
            cs.wait_stream(s)
            issue_copy(0)
            for i in range(K):
                k = i % 2
                if i + 1 < K:
                    issue_copy(1 - k)
                s.wait_event(copied[k])
                s.wait_event(results_read[k])  # results of step i-2 have left buffer set k
                o, gs = rbufs[k]
                r = step(Xd[k], bufs=rbufs[k]) if args.infer else step(Xd[k], doutd[k], bufs=rbufs[k])
                consumed[k].record(s)
                results_ready[k].record(s)
                with torch.cuda.stream(ds):
                    ds.wait_event(results_ready[k])
                    outh[own_rows].copy_(o[own_rows], non_blocking=True)
                    if not args.infer:
                        dxh.copy_(r[own_rows], non_blocking=True)
                        for name in wkeys:
                            dwh[name].copy_(gs[name], non_blocking=True)
                    results_read[k].record(ds)
            s.wait_stream(ds)

        e2e_run(2)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        s = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        e2e_run(args.steps)
        e1.record(s)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ems], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": g.num_edges * args.steps / (ems / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": ems / args.steps,
               "path": "paper_2412_04747_b200.Layer forward/backward (C-ABI); per step H2D of X and dout from pinned "
                       "host memory (double-buffered on a copy stream: step i+1's copy overlaps step i), D2H of the "
                       "step's results (the owned output rows, the owned dX rows and every weight gradient) on a "
                       "second copy stream; the next step waits until the results have been read"}

    # ---- roofline of the dominant kernel
    peaks = load_peaks()
    gi = G.info()
    U, E = gi["num_pairs"], gi["num_edges"]
    bsz = 2 if dtype == "bf16" else 4
    spmm = rgat_spmm_on(args)
    UD = dst_rel_pairs(g) if model == "rgat" else 0
    alg = algorithmic_bytes(model, dtype, g.num_nodes, E, U, UD, g.num_rels, g.num_node_types, d, d, spmm)
    alg = adjust_for_fusions(alg, prof, U, g.num_nodes, d, bsz)
    if world == 1 and not args.no_compact and model in ("hgt", "rgat"):
        alg = adjust_for_single(alg, model, E, U, single_edge_pairs(g), d, bsz, spmm)
    roofline = roofline_block(alg, prof, args.steps, ms_per_step, peaks, model, dtype, g.num_nodes, E, U, d,
                              t_fwd, t_bwd, args.infer)
    kernels = roofline.pop("_kernels")
    if roofline.get("kernel") and world == 1 and not args.no_ncu and not args.cuda_graph:
        tr = ncu_traffic_in_run(args, roofline["kernel"])
        if tr is not None:
            ms_k = roofline["ms_per_step"]
            roofline["traffic"] = int(tr["bytes_per_step"])
            roofline["traffic_frac"] = tr["bytes_per_step"] / (ms_k / 1e3) / 1e9 / peaks["hbm_gbs"]
            roofline["traffic_note"] = ("ncu DRAM read+write bytes per step of this label, cold-cache serialised "
                                        "replays; traffic_frac = these bytes / the live event time / peak")
            roofline["traffic_how"] = tr["how"]
            roofline["traffic_source_hash"] = tr["source_hash"]

    gi = G.info()
    memory = {"graph_index_bytes": int(gi["device_bytes"]), "saved_bytes": int(layer.saved.numel()),
              "scratch_bytes": int(layer.scratch.numel()),
              "features_bytes": int(X_full.numel() * X_full.element_size() + out.numel() * 4 +
                                    (0 if args.infer else dout.numel() * 4 + grads["dX"].numel() * 4)),
              "weights_bytes": int(sum(v.numel() * v.element_size() for v in w.values())),
              "peak_allocated_bytes": int(torch.cuda.max_memory_allocated(dev)),
              "note": "saved = forward->backward activations (compact: U rows; vanilla: E rows), scratch = "
                      "per-call temporaries; the graph handle also holds the work lists and cached tile plans"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.infer:
        if cfg.get("heads", 1) == 1 and not args.no_compact:
            # D5: nproc threads on the full graph; one thread on an in-edge sample of ~E / nproc edges
            cpu = cpu_oracle_grouped(g, model, inp, Gh)
            st = cpu_oracle_grouped(g, model, inp, Gh, max_edges=g.num_edges // max(1, os.cpu_count() or 1),
                                    threads=1)
            cpu["single_thread"] = {k: st[k] for k in ("value", "unit", "cores", "sample")}
        else:  # heads > 1: the per-edge numpy oracle (the grouped C oracle is one-head)
            cpu = cpu_oracle_sample(g, model, inp, Gh, target_s=args.cpu_seconds)
            cpu["single_thread"] = single_thread(lambda t: cpu_oracle_sample(g, model, inp, Gh, target_s=t),
                                                 args.cpu_seconds / 3)

    exchange = None
    if world > 1:  # bytes of variant X vs variant P per rank, and the one run
        u_glob = int(np.unique(g.rel.astype(np.int64) * g.num_nodes + g.src).size)
        exchange = rgnn.exchange_bytes(model, dtype, d, d, g.num_nodes, u_glob, cfg.get("heads", 1))
        exchange["how"] = ("library-owned NCCL (rgnn_comm): in-place all-gather of X by owner broadcasts on the "
                           "library's stream, chunk-pipelined with the pair GEMM; dX reduced onto the owners, dW "
                           "all-reduced, inside rgnn_layer_forward / rgnn_layer_backward")
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step,
            "ms_per_step_median": float(np.median(per_step_timed)) if per_step_timed else None,
            "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": dtype, "data": "synthetic",
            "config": {"workload": f"{cfg['graph']}-shaped {model.upper()} layer fwd+bwd, hidden {d} "
                                   f"(BASELINE.json configs[{cfg['baseline']}])",
                       "graph": cfg["graph"], "layer": model, "d_in": d, "d_out": d,
                       "nodes": g.num_nodes, "edges": int(g.num_edges), "pairs": int(info["num_pairs"]) if world == 1 else None,
                       "relations": g.num_rels, "node_types": g.num_node_types,
                       "compaction_ratio": info["compaction_ratio"], "max_in_degree": info["max_in_degree"],
                       "max_pair_degree": info["max_pair_degree"],
                       "parallelism": f"dst-partition x{world}" if world > 1 else "single GPU",
                       "l2": "inputs larger than L2 (X %.2f GB, pair table %.2f GB, index arrays %.2f GB)" % (
                           g.num_nodes * d * (2 if dtype == 'bf16' else 4) / 1e9,
                           info["num_pairs"] * 2 * d * (2 if dtype == 'bf16' else 4) / 1e9,
                           g.num_edges * 4 * 9 / 1e9),
                       "gemm_impl": ["auto (bf16 -> tcgen05)", "simt", "tcgen05"][args.gemm_impl],
                       "materialization": "vanilla (row per edge)" if args.no_compact else "compact (row per (rel, src) pair)",
                       "reorder": not args.no_reorder, "heads": cfg.get("heads", 1), "mode": "inference (forward only)" if args.infer else "training (forward + backward)",
                       "cuda_graph": bool(use_graph), "a_dst": args.a_dst if args.a_dst is not None else 0.8,
                       "exchange": exchange},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clocks, "remeasured_for_clocks": remeasured, "memory": memory, "kernels": kernels,
            "kernel_timing": KERNEL_TIMING[bool(args.profile_in_timed) and not use_graph],
        }
        print(json.dumps(line))
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


# ----------------------------------------------------------------- F4 training step
TRAIN_LR = 1e-3
LABEL_SEED, LABELLED_FRAC = 5, 1.0


def train_bytes(model, dtype, N, E, U, R, T, d, layers, num_params, UD=0, rgat_spmm=True):
    """Algorithmic bytes per training step: every layer kernel once per layer (the dX kernels of
    layer 1 are pruned: its input is data), plus the F4 kernels."""
    b = 2 if dtype == "bf16" else 4
    per = algorithmic_bytes(model, dtype, N, E, U, UD, R, T, d, d, rgat_spmm)
    dx = {"gemm_pairs_dx", "gemm_nodes_dx", "seg_reduce_rows", "gemm_selfloop_dx", "pair_bwd_fused"}
    out = {k: v * (layers - 1 if k in dx else layers) for k, v in per.items()}
    if b == 2:  # bf16: layers 2.. run the fused A8 kernel (dX rows + dW); only layer 1 (no dX) runs wgrad_pairs
        out["wgrad_pairs"] = per["wgrad_pairs"]
    out["relu_fwd"] = (layers - 1) * N * d * (4 + b)
    out["relu_bwd"] = (layers - 1) * N * d * 12
    out["nll_loss"] = N * d * 8 + N * 4
    out["sgd_update"] = num_params * (4 + 4 + 4 + (b if b == 2 else 0))
    return out


def cpu_train_sample(cfg, layers, target_s=15.0):
    """The fp64 oracle's training step (oracle/train.py, as it stands) on the same generator at a
    reduced scale, grown until one step takes a few seconds; edges/s = layers * E / step time."""
    from oracle import train as OT
    from synth import stack_inputs, random_labels
    try:
        from threadpoolctl import threadpool_info
        threads = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        threads = os.cpu_count() or 1
    trained = {"rgcn": ("W", "W0"), "rgat": ("W", "a", "b"), "hgt": ("Wk", "Wq", "Wv", "Watt", "Wmsg")}[cfg["model"]]
    scale, tot_t, tot_e = 1e-3, 0.0, 0
    while True:
        g = config_graph(cfg["graph"], seed=1, scale=scale)
        ps = stack_inputs(cfg["model"], g, cfg["d"], layers)
        X = ps[0].pop("X")
        y = random_labels(g.num_nodes, cfg["d"], seed=LABEL_SEED)
        t = time.perf_counter()
        OT.train_step(cfg["model"], g, X, ps, y, TRAIN_LR, trained)
        dt = time.perf_counter() - t
        tot_t += dt
        tot_e += layers * g.num_edges
        if tot_t >= 0.5 * target_s or scale >= 1.0:
            break
        scale = min(1.0, scale * max(2.0, min(8.0, 0.5 * target_s / max(dt, 1e-3))))
    return {"value": tot_e / tot_t, "unit": UNIT, "cores": int(threads), "kind": "oracle", "cpu_model": cpu_model(),
            "nproc": os.cpu_count(),
            "sample": f"fp64 numpy oracle {layers}-layer {cfg['model'].upper()} training step (oracle/train.py) on the "
                      f"{cfg['graph']} generator at growing scales up to {scale:g} ({g.num_edges} edges); "
                      f"{tot_e} layer-edges in {tot_t:.1f} s", "seconds": tot_t}


def run_train(args, cfg, world, rank, local_rank):
    """F4: one step = `layers` stacked layers forward (ReLU between), NLL loss vs a random label
    tensor, backward through the stack, SGD update of every weight.  value = layers * E
    edges per step / step time (each layer processes every edge forward and backward)."""
    import torch
    from paper_2412_04747_b200 import Graph, Stack, rgnn
    from synth import stack_inputs, random_labels
    if world > 1:
        raise SystemExit("training-step configs run on one GPU (the partitioned path is the layer bench)")
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    layers = cfg["layers"]
    g = config_graph(cfg["graph"], seed=1, a_dst=args.a_dst)
    model, d, dtype = cfg["model"], cfg["d"], cfg["dtype"]
    G = Graph.from_hetero(g, device=dev, compact=not args.no_compact)
    info = G.info()
    ps = stack_inputs(model, g, d, layers)
    Xh64 = ps[0].pop("X")
    td = torch.float32 if dtype == "f32" else torch.bfloat16
    st = Stack(G, model, d, [{k: torch.tensor(v) for k, v in p.items()} for p in ps], dtype=dtype,
               reorder=not args.no_reorder)
    X = torch.tensor(Xh64.astype(np.float32), device=dev).to(td)
    y = random_labels(g.num_nodes, d, seed=LABEL_SEED, labelled_frac=LABELLED_FRAC)
    nl = int((y >= 0).sum())
    labels = torch.tensor(y, device=dev)

    def step(Xd, yd):
        return st.train_step(Xd, yd, nl, TRAIN_LR)

    for _ in range(args.warmup):
        step(X, labels)
    torch.cuda.synchronize()
    graph = None
    if args.cuda_graph:  # launch-bound small graphs: replay one captured training step
        cs = torch.cuda.Stream()
        cs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cs):
            step(X, labels)
        torch.cuda.current_stream().wait_stream(cs)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step(X, labels)
        torch.cuda.synchronize()
    sampler = ClockSampler(local_rank)
    sampler.start()
    time.sleep(0.15)

    prof_on = [bool(args.profile_in_timed)]

    def timed(K, use_graph=False):
        torch.cuda.synchronize()
        rgnn.profile_reset()
        rgnn.profile_enable(not use_graph and prof_on[0])
        n0 = rgnn.launch_count()
        s = torch.cuda.current_stream()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
        t0 = time.time()
        ev[0].record(s)
        for i in range(K):
            if use_graph:
                graph.replay()
            else:
                step(X, labels)
            ev[i + 1].record(s)
        torch.cuda.synchronize()
        t1 = time.time()
        launches = rgnn.launch_count() - n0
        prof = rgnn.profile_read()
        rgnn.profile_enable(False)
        per = [ev[i].elapsed_time(ev[i + 1]) for i in range(K)]
        return ev[0].elapsed_time(ev[K]), per, launches, prof, t0, t1

    use_graph = graph is not None
    ms, per, launches, prof, t0, t1 = timed(args.steps, use_graph)
    time.sleep(0.12)
    clocks = sampler.summary(t0, t1)
    remeasured = False
    if set(clocks["reasons"]) & BAD_REASONS:
        remeasured = True
        ms, per, launches, prof, t0, t1 = timed(args.steps, use_graph)
        time.sleep(0.12)
        clocks = sampler.summary(t0, t1)
    if use_graph or not args.profile_in_timed:  # per-kernel attribution: a second timed pass with launch events
        prof_on[0] = True
        _, _, launches, prof, _, _ = timed(args.steps, False)
        prof_on[0] = bool(args.profile_in_timed)
    sampler.stop()
    loss_now = float(st.nll.loss.item())
    ms_per_step = ms / args.steps
    value = layers * g.num_edges * args.steps / (ms / 1e3)

    e2e = None
    if not args.no_e2e:
        Xh = X.cpu().pin_memory()
        yh = labels.cpu().pin_memory()
        lossh = torch.empty(1, dtype=torch.float32).pin_memory()
        Xd = [torch.empty_like(X) for _ in range(2)]
        yd = [torch.empty_like(labels) for _ in range(2)]
        cs = torch.cuda.Stream(device=dev)
        copied = [torch.cuda.Event() for _ in range(2)]
        consumed = [torch.cuda.Event() for _ in range(2)]

        def issue_copy(k):
            with torch.cuda.stream(cs):
                cs.wait_event(consumed[k])
                Xd[k].copy_(Xh, non_blocking=True)
                yd[k].copy_(yh, non_blocking=True)
                copied[k].record(cs)

        def e2e_run(K):
            s = torch.cuda.current_stream()
            cs.wait_stream(s)
            issue_copy(0)
            for i in range(K):
                k = i % 2
                if i + 1 < K:
                    issue_copy(1 - k)
                s.wait_event(copied[k])
                lossh.copy_(step(Xd[k], yd[k]), non_blocking=True)
                consumed[k].record(s)

        e2e_run(2)
        torch.cuda.synchronize()
        s = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        e2e_run(args.steps)
        e1.record(s)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1)
        e2e = {"value": layers * g.num_edges * args.steps / (ems / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(Xh.numel() * Xh.element_size() + yh.numel() * 4),
               "d2h_bytes_per_step": 4, "ms_per_step": ems / args.steps,
               "path": "paper_2412_04747_b200.Stack.train_step (C-ABI); per step H2D of X and the labels from pinned "
                       "host memory (double-buffered on a copy stream), D2H of the loss"}

    peaks = load_peaks()
    U, E = info["num_pairs"], info["num_edges"]
    nparams = sum(m.numel() for ms_ in st.master for m in ms_.values())
    spmm = rgat_spmm_on(args)
    UD = dst_rel_pairs(g) if model == "rgat" else 0
    alg = train_bytes(model, dtype, g.num_nodes, E, U, g.num_rels, g.num_node_types, d, layers, nparams, UD, spmm)
    alg = adjust_for_fusions(alg, prof, U * (layers - 1), g.num_nodes * (layers - 1), d, 2 if dtype == "bf16" else 4)
    if not args.no_compact and model in ("hgt", "rgat"):
        one = adjust_for_single({k: 0 for k in alg}, model, E, U, single_edge_pairs(g), d,
                                2 if dtype == "bf16" else 4, spmm)
        alg = {k: v + layers * one.get(k, 0) for k, v in alg.items()}
    tot_ms = sum(x["ms"] for x in prof.values())
    kernels = {k: {"launches_per_step": v["launches"] / args.steps, "ms_per_step": v["ms"] / args.steps,
                   "share": v["ms"] / max(tot_ms, 1e-9)} for k, v in prof.items()}
    for k in kernels:
        if k in alg and alg[k]:
            kernels[k]["algorithmic_bytes_per_step"] = int(alg[k])
            kernels[k]["achieved_gbs"] = alg[k] / (kernels[k]["ms_per_step"] / 1e3) / 1e9
    dom = max((k for k in prof if k in alg), key=lambda k: prof[k]["ms"], default=None)
    roofline = None
    if dom is not None:
        ms_k = kernels[dom]["ms_per_step"]
        achieved = alg[dom] / (ms_k / 1e3) / 1e9
        ran = sum(v for k, v in alg.items() if k in prof)  # only the labels that launched
        roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                    "frac": achieved / peaks["hbm_gbs"], "traffic": None, "peak_source": peaks["source"],
                    "algorithmic_bytes_per_step": int(alg[dom]), "launches_per_step": kernels[dom]["launches_per_step"],
                    "ms_per_step": ms_k, "step_algorithmic_gb": ran / 1e9,
                    "step_achieved_gbs": ran / (ms_per_step / 1e3) / 1e9,
                    "note": "bytes and time per step of the kernel label (all its launches in one step, both layers)"}
    cpu = None
    if not args.no_cpu_baseline:
        cpu = cpu_train_sample(cfg, layers, target_s=args.cpu_seconds)
        cpu["single_thread"] = single_thread(lambda t: cpu_train_sample(cfg, layers, target_s=t), args.cpu_seconds / 3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "ms_per_step_median": float(np.median(per)),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": dtype, "data": "synthetic",
        "config": {"workload": f"{cfg['graph']}-shaped {layers}-layer {model.upper()} training step, hidden {d} "
                               f"(BASELINE.json configs[{cfg['baseline']}]): layers + ReLU + NLL loss vs random labels "
                               f"+ backward + SGD; value counts E edges per layer",
                   "graph": cfg["graph"], "layer": model, "layers": layers, "d": d, "nodes": g.num_nodes,
                   "edges": int(g.num_edges), "pairs": int(U), "relations": g.num_rels,
                   "node_types": g.num_node_types, "compaction_ratio": info["compaction_ratio"],
                   "labelled_rows": nl, "lr": TRAIN_LR, "loss_after_timed_steps": loss_now,
                   "parallelism": "single GPU", "l2": "flush: none; working set %.2f GB %s L2 (126 MB)" % (
                       sum(alg.values()) / 1e9 / max(1, layers), ">" if sum(alg.values()) > 126e6 * layers else "~"),
                   "materialization": "vanilla (row per edge)" if args.no_compact else "compact (row per (rel, src) pair)",
                   "reorder": not args.no_reorder, "mode": "training (2-layer step incl. loss and SGD)",
                   "cuda_graph": use_graph, "a_dst": args.a_dst if args.a_dst is not None else 0.8},
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
        "clocks": clocks, "remeasured_for_clocks": remeasured, "kernels": kernels,
        "kernel_timing": KERNEL_TIMING[bool(args.profile_in_timed) and not use_graph],
        "memory": {"graph_index_bytes": int(info["device_bytes"]),
                   "saved_bytes": int(sum(l.saved.numel() for l in st.layers)),
                   "scratch_bytes": int(sum(l.scratch.numel() for l in st.layers)),
                   "peak_allocated_bytes": int(torch.cuda.max_memory_allocated(dev))},
    }
    print(json.dumps(line))


def run_reference(args, cfg, world, rank):
    """Reference arm of this tier: the fp64 oracle as it stands on the host cores; each step is
    a bounded sample of the workload (in-edge subgraph of random destinations)."""
    if rank != 0:
        return
    if cfg.get("layers", 1) > 1:
        vals, secs, edges = [], 0.0, 0
        per_step = max(2.0, 60.0 / max(1, args.steps + args.warmup))
        for i in range(args.steps):
            r = cpu_train_sample(cfg, cfg["layers"], target_s=per_step)
            secs += r["seconds"]
            edges += r["value"] * r["seconds"]
        value = edges / secs
        print(json.dumps({"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
                          "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                          "data": "synthetic",
                          "config": {"workload": f"{cfg['graph']}-shaped {cfg['layers']}-layer {cfg['model'].upper()} "
                                                 "training step, bounded sample per step", "graph": cfg["graph"]},
                          "cpu_baseline": {"value": value, "unit": UNIT, "cores": r["cores"], "kind": "oracle",
                                           "sample": r["sample"]},
                          "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
        return
    g = config_graph(cfg["graph"], seed=1)
    model, d = cfg["model"], cfg["d"]
    inp = layer_inputs(model, g, d, d)
    if cfg["dtype"] == "bf16":
        inp = {k: (round_bf16(v) if k not in ("mu",) else v) for k, v in inp.items()}
    Gh = upstream_grad(g.num_nodes, d)
    # each step: the grouped oracle on all host cores over an in-edge sample sized to ~per_step seconds
    # (rate measured on a first small sample); the whole --steps/--warmup run stays within a few minutes
    per_step = max(2.0, 120.0 / max(1, args.steps + args.warmup))
    probe = cpu_oracle_grouped(g, model, inp, Gh, max_edges=max(1, g.num_edges // 64), seed=999)
    step_edges = int(min(g.num_edges, probe["value"] * per_step))
    for i in range(args.warmup):
        cpu_oracle_grouped(g, model, inp, Gh, max_edges=max(1, step_edges // 4), seed=100 + i)
    vals, secs, edges = [], 0.0, 0
    last = None
    for i in range(args.steps):
        r = cpu_oracle_grouped(g, model, inp, Gh, max_edges=step_edges, seed=i)
        vals.append(r["value"])
        secs += r["seconds"]
        edges += r["value"] * r["seconds"]
        last = r
    value = edges / secs
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"{cfg['graph']}-shaped {model.upper()} layer fwd+bwd, hidden {d} "
                                   f"(BASELINE.json configs[{cfg['baseline']}]) — bounded sample per step",
                       "graph": cfg["graph"], "layer": model, "d_in": d, "d_out": d},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": last["cores"], "kind": "oracle",
                             "sample": last["sample"]},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
