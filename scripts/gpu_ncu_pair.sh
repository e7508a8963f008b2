python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
python bench.py --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/e2e_bench_mag_hgt.json
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_hgt_bwd_pair|k_hgt_bwd_dst|k_hgt_fwd' --launch-skip 18 --launch-count 6 -o gpurun_out/prof_trav python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof_trav.log 2>&1
