# final verification + refreshed bench lines after the fused-A8 ring (round 1)
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
mkdir -p gpurun_out/fin2
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -2 > gpurun_out/fin2/pytest_gpu.txt; cat gpurun_out/fin2/pytest_gpu.txt
python bench.py 2>&1 | tail -1 > gpurun_out/fin2/bench_mag_hgt.json
for c in mag_rgat am_rgat am_rgat_train bgs_rgat mag_hgt_train; do
  python bench.py --config $c --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/fin2/bench_$c.json
done





ls gpurun_out/fin2
