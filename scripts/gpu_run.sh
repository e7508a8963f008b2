#!/bin/bash
# One driver for the GPU-box tasks of this repo (run under /usr/local/graft/bin/gpurun from the repo root):
#   bash scripts/gpu_run.sh verify            build, full GPU suite, smoke, default bench line
#   bash scripts/gpu_run.sh ab CONFIG VAR...  one bench line per environment assignment (A/B of a switch),
#                                             e.g. ab mag_hgt RGNN_PAIR_WS=1 RGNN_PAIR_WS=0
#   bash scripts/gpu_run.sh evidence          every bench line (profiles/rNN_bench_*.json material), the ncu
#                                             launch list of the default bench
#   bash scripts/gpu_run.sh ablation          F1 C/R ablation runs (scripts/ablation_table.py summarises them)
#   bash scripts/gpu_run.sh ncu KERNEL_REGEX [CONFIG]   ncu --set full of the matching kernels of one step
#   bash scripts/gpu_run.sh abhead CONFIG...  HEAD (a clean checkout in ab_head/, made by scripts/mk_ab_head.sh)
#                                             against the working tree, interleaved, twice per config
# Outputs go to gpurun_out/$TAG/ (TAG defaults to the task name).
set -u
task=${1:-verify}; shift || true
out=gpurun_out/${TAG:-$task}
mkdir -p "$out"
build() { python -c "import __graft_entry__ as g; g.build()" > "$out/build.log" 2>&1 || { tail -30 "$out/build.log"; exit 1; }; }
summ() {  # summ LOG LABEL: ms/step and the per-kernel times of a bench line
  python - "$1" "$2" <<'PY'
import json, sys
ls = [x for x in open(sys.argv[1]) if x.startswith("{")]
if not ls:
    print(sys.argv[2], "no result"); sys.exit()
j = json.loads(ls[-1])
print(sys.argv[2], round(j["ms_per_step"], 3), {k: round(v["ms_per_step"], 3) for k, v in j.get("kernels", {}).items()
                                                if v["ms_per_step"] > 0.02})
PY
}
case "$task" in
  verify)
    build
    timeout 1800 python -m pytest tests -m gpu -q > "$out/pytest.log" 2>&1; tail -3 "$out/pytest.log"
    python -c "import __graft_entry__ as g; g.smoke()" > "$out/smoke.log" 2>&1; tail -2 "$out/smoke.log"
    timeout 900 python bench.py > "$out/bench.json" 2> "$out/bench.err"; summ "$out/bench.json" default
    ;;
  ab)
    build
    cfg=$1; shift
    for v in "$@"; do
      env $v timeout 300 python bench.py --config "$cfg" --no-cpu-baseline --no-ncu --no-e2e --steps 20 \
        > "$out/${cfg}_${v//[^A-Za-z0-9_]/_}.json" 2>&1
      summ "$out/${cfg}_${v//[^A-Za-z0-9_]/_}.json" "$cfg $v"
    done
    ;;
  evidence)
    build
    timeout 1800 python -m pytest tests -m gpu -q > "$out/pytest.log" 2>&1; tail -3 "$out/pytest.log"
    python -c "import __graft_entry__ as g; g.smoke()" > "$out/smoke.log" 2>&1; tail -2 "$out/smoke.log"
    timeout 900 python bench.py > "$out/bench_mag_hgt.json" 2> "$out/bench_mag_hgt.err"; summ "$out/bench_mag_hgt.json" mag_hgt
    for c in ${CONFIGS:-am_rgat mag_rgat wikikg2_rgcn am_hgt mag_hgt_f32 mag_hgt_h8 biokg_hgt mag_hgt_train am_rgat_train}; do
      timeout 900 python bench.py --config "$c" --no-ncu > "$out/bench_$c.json" 2> "$out/bench_$c.err"; summ "$out/bench_$c.json" "$c"
    done
    for c in ${GRAPH_CONFIGS:-aifb_rgat bgs_rgat mutag_rgat fb15k_rgcn aifb_hgt aifb_rgat_train bgs_rgat_train}; do
      timeout 900 python bench.py --config "$c" --cuda-graph --no-ncu > "$out/bench_${c}_graph.json" 2> "$out/bench_${c}_graph.err"
      summ "$out/bench_${c}_graph.json" "$c graph"
    done
    timeout 900 python bench.py --impl reference > "$out/bench_reference.json" 2>&1; tail -c 300 "$out/bench_reference.json"; echo
    timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file "$out/launches_mag_hgt.csv" python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-ncu --no-e2e > /dev/null 2>&1  # 5 launches per step kernel (launch_summary.py CSV 5)
    # compute-sanitizer is closed on the GPU pool (round 2); the last memcheck log is profiles/r02_memcheck_gpu_suite.log
    ;;
  ablation)
    build
    for c in ${CONFIGS:-mag_hgt am_hgt aifb_hgt am_rgat aifb_rgat mag_rgat}; do
      for mode in "" "--infer"; do
        tag=$(echo "$c$mode" | tr -d ' -')
        python bench.py --config $c $mode --no-cpu-baseline --no-e2e 2>&1 | tail -1 > "$out/${tag}_CR.json"
        python bench.py --config $c $mode --no-reorder --no-cpu-baseline --no-e2e 2>&1 | tail -1 > "$out/${tag}_C.json"
        python bench.py --config $c $mode --no-compact --no-cpu-baseline --no-e2e 2>&1 | tail -1 > "$out/${tag}_R.json"
        python bench.py --config $c $mode --no-compact --no-reorder --no-cpu-baseline --no-e2e 2>&1 | tail -1 > "$out/${tag}_U.json"
      done
    done
    ;;
  abhead)
    build
    # HEAD_DEFINES: RGNN_DEFINES of the ab_head build (a build-time variant instead of another commit)
    (cd ab_head && RGNN_DEFINES="${HEAD_DEFINES:-}" python -c "import __graft_entry__ as g; g.build()" > "../$out/build_head.log" 2>&1) || { tail -30 "$out/build_head.log"; exit 1; }
    for cfg in "$@"; do
      for i in 1 2; do
        (cd ab_head && timeout 300 python bench.py --config "$cfg" --no-cpu-baseline --no-ncu --no-e2e --steps 20 \
          > "../$out/${cfg}_head$i.json" 2>&1); summ "$out/${cfg}_head$i.json" "$cfg HEAD"
        timeout 300 python bench.py --config "$cfg" --no-cpu-baseline --no-ncu --no-e2e --steps 20 \
          > "$out/${cfg}_new$i.json" 2>&1; summ "$out/${cfg}_new$i.json" "$cfg NEW "
      done
    done
    ;;
  ncu)
    build
    timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$1" -o "$out/ncu" \
      python bench.py --config "${2:-mag_hgt}" --no-cpu-baseline --no-ncu --no-e2e --steps 1 --warmup 1 > "$out/ncu.log" 2>&1
    tail -2 "$out/ncu.log"
    ncu -i "$out/ncu.ncu-rep" --page details --csv > "$out/details.csv" 2>/dev/null
    python scripts/ncu_summary.py "$out/details.csv" > "$out/summary.txt"; head -60 "$out/summary.txt"
    ncu -i "$out/ncu.ncu-rep" --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct,smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct,smsp__warp_issue_stalled_mio_throttle_per_warp_active.pct,l1tex__t_bytes_pipe_lsu_mem_global_op_ld.sum,sm__warps_active.avg.pct_of_peak_sustained_active > "$out/raw.csv" 2>/dev/null
    # the report itself only when small enough to travel back (gpurun copies <= 64 MiB)
    [ "$(stat -c %s "$out/ncu.ncu-rep")" -gt 40000000 ] && rm -f "$out/ncu.ncu-rep"
    ;;
  *) echo "unknown task $task"; exit 2 ;;
esac
