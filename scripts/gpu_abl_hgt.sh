python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
mkdir -p gpurun_out/abl
for c in aifb_hgt am_hgt; do
  for mode in "" "--infer"; do
    tag=$(echo "$c$mode" | tr -d ' -')
    python bench.py --config $c $mode --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/abl/${tag}_CR.json
    python bench.py --config $c $mode --no-compact --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/abl/${tag}_R.json
  done
done
timeout 1500 python -m pytest tests -q -x -m "gpu and not slow" 2>&1 | tail -3
python bench.py --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/bench_mag_hgt.json
