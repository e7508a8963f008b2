# round profile refresh: bench lines (all configs), ncu launch list and one ncu --set full of the step's kernels
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
python bench.py 2>&1 | tail -1 > gpurun_out/prof_bench_mag_hgt.json
for c in mag_hgt_f32 mag_rgat am_rgat am_hgt aifb_rgat bgs_rgat wikikg2_rgcn; do
  python bench.py --config $c --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/prof_bench_$c.json
done
python bench.py --config aifb_rgat --cuda-graph --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/prof_bench_aifb_rgat_graph.json
python bench.py --impl reference --steps 3 --warmup 3 2>&1 | tail -1 > gpurun_out/prof_bench_reference.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:'k_hgt|k_gemm|k_wgrad|k_seg|k_merge' --launch-skip 60 --launch-count 20 -o gpurun_out/prof_full python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof_full.log 2>&1
