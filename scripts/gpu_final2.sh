# final verification + refreshed bench lines after the fused-A8 ring (round 1)
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
mkdir -p gpurun_out/fin2
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -2 > gpurun_out/fin2/pytest_gpu.txt; cat gpurun_out/fin2/pytest_gpu.txt
python bench.py 2>&1 | tail -1 > gpurun_out/fin2/bench_mag_hgt.json
for c in mag_hgt_h8 mag_rgat am_rgat am_hgt wikikg2_rgcn biokg_hgt mag_hgt_train am_rgat_train bgs_rgat; do
  python bench.py --config $c --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/fin2/bench_$c.json
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin2/launches_mag_hgt.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/fin2/launches_mag_hgt.csv 5 > gpurun_out/fin2/launches_mag_hgt.txt
timeout 900 ncu --set full --clock-control none -k regex:'k_gemm|k_wgrad|k_pair_bwd' --launch-skip 15 --launch-count 5 -o gpurun_out/fin2/ncu_gemm_mag_hgt python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fin2/ncu_gemm.log 2>&1
ncu -i gpurun_out/fin2/ncu_gemm_mag_hgt.ncu-rep --page details --csv > gpurun_out/fin2/ncu_gemm_mag_hgt.details.csv 2>/dev/null
rm -f gpurun_out/fin2/ncu_gemm_mag_hgt.ncu-rep
ls gpurun_out/fin2
