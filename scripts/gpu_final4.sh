python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out/fin4
for c in am_hgt am_rgat am_rgat_train mag_rgat; do
  python bench.py --config $c --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/fin4/bench_$c.json
done
python bench.py 2>&1 | tail -1 > gpurun_out/fin4/bench_mag_hgt.json
