# round-1 final profile refresh: smoke, bench lines of every config, reference arm, ncu launch list and
# ncu --set full of the traversal kernels (mag HGT + AM RGAT + wikikg2 RGCN)
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
mkdir -p gpurun_out/fin
timeout 1500 python -m pytest tests -q -x -m gpu 2>&1 | tail -2 > gpurun_out/fin/pytest_gpu.txt
python bench.py 2>&1 | tail -1 > gpurun_out/fin/bench_mag_hgt.json
for c in mag_hgt_f32 mag_hgt_h8 mag_rgat am_rgat am_hgt bgs_rgat wikikg2_rgcn biokg_hgt; do
  python bench.py --config $c --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/fin/bench_$c.json
done
for c in aifb_rgat mutag_rgat fb15k_rgcn aifb_hgt; do
  python bench.py --config $c --no-cpu-baseline --cuda-graph 2>&1 | tail -1 > gpurun_out/fin/bench_${c}_graph.json
done
for c in mag_hgt_train am_rgat_train; do python bench.py --config $c --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/fin/bench_$c.json; done
for c in aifb_rgat_train bgs_rgat_train; do python bench.py --config $c --no-cpu-baseline --cuda-graph 2>&1 | tail -1 > gpurun_out/fin/bench_${c}_graph.json; done
python bench.py --impl reference --steps 3 --warmup 3 2>&1 | tail -1 > gpurun_out/fin/bench_reference.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin/launches_mag_hgt.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/fin/launches_mag_hgt.csv 5 > gpurun_out/fin/launches_mag_hgt.txt
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_hgt_(fwd|bwd)' --launch-skip 27 --launch-count 9 -o gpurun_out/fin/ncu_trav_mag_hgt python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fin/ncu_trav_mag_hgt.log 2>&1
timeout 1200 ncu --set full --clock-control none -k regex:'k_gemm|k_wgrad|k_seg_reduce' --launch-skip 21 --launch-count 7 -o gpurun_out/fin/ncu_gemm_mag_hgt python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fin/ncu_gemm_mag_hgt.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:'k_rgat_(fwd|bwd)' --launch-skip 18 --launch-count 6 -o gpurun_out/fin/ncu_trav_am_rgat python bench.py --config am_rgat --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fin/ncu_trav_am_rgat.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:'k_rgcn_(fwd|bwd)' --launch-skip 15 --launch-count 5 -o gpurun_out/fin/ncu_trav_wikikg2_rgcn python bench.py --config wikikg2_rgcn --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fin/ncu_trav_wikikg2_rgcn.log 2>&1
# reports -> text (details + raw csv); keep only the mag HGT traversal report (gpurun_out is capped at 64 MiB)
for r in ncu_trav_mag_hgt ncu_gemm_mag_hgt ncu_trav_am_rgat ncu_trav_wikikg2_rgcn; do
  if [ -f gpurun_out/fin/$r.ncu-rep ]; then
    ncu -i gpurun_out/fin/$r.ncu-rep --page details --csv > gpurun_out/fin/$r.details.csv 2>/dev/null
    ncu -i gpurun_out/fin/$r.ncu-rep --page raw --csv > gpurun_out/fin/$r.raw.csv 2>/dev/null
    [ "$r" != ncu_trav_mag_hgt ] && rm -f gpurun_out/fin/$r.ncu-rep
  fi
done
ls -la gpurun_out/fin; du -sh gpurun_out
