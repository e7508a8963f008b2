# F1: C/R ablation (tab:optimizations shape) on the bench configs, training and inference.
# C = compact + reordering off, R = vanilla + reordered, CR = both (default), U = neither.
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1500 python -m pytest tests/test_gpu_layers.py -q -x -k "no_reorder" 2>&1 | tail -3
mkdir -p gpurun_out/abl
for c in ${CONFIGS:-mag_hgt am_hgt aifb_hgt am_rgat aifb_rgat mag_rgat}; do
  for mode in "" "--infer"; do
    tag=$(echo "$c$mode" | tr -d ' -')
    python bench.py --config $c $mode --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/abl/${tag}_CR.json
    python bench.py --config $c $mode --no-reorder --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/abl/${tag}_C.json
    python bench.py --config $c $mode --no-compact --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/abl/${tag}_R.json
    python bench.py --config $c $mode --no-compact --no-reorder --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/abl/${tag}_U.json
  done
done
echo ablation-done
