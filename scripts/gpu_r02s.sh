# round-2 closing evidence: full GPU suite, smoke, every bench line (profiles/r02_bench_*.json),
# the ncu launch list of the default bench, compute-sanitizer memcheck over a GPU-suite subset
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02s_build.log 2>&1 || { tail -30 gpurun_out/r02s_build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02s_pytest.log 2>&1; tail -3 gpurun_out/r02s_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02s_smoke.log 2>&1; tail -2 gpurun_out/r02s_smoke.log
mkdir -p gpurun_out/r02s
timeout 900 python bench.py > gpurun_out/r02s/bench_mag_hgt.json 2>gpurun_out/r02s/bench_mag_hgt.err; tail -c 300 gpurun_out/r02s/bench_mag_hgt.json; echo
for c in am_rgat mag_rgat wikikg2_rgcn am_hgt mag_hgt_f32 mag_hgt_h8 biokg_hgt mag_hgt_train am_rgat_train; do
  timeout 900 python bench.py --config $c --no-ncu > gpurun_out/r02s/bench_$c.json 2>gpurun_out/r02s/bench_$c.err
  python -c "import json,sys; l=[x for x in open('gpurun_out/r02s/bench_$c.json') if x.startswith('{')][-1]; j=json.loads(l); print('$c', round(j['ms_per_step'],3), round(j['value']/1e9,3), j['roofline'].get('kernel'), round(j['roofline'].get('frac') or 0,3), j['roofline'].get('step_d4_frac'))"
done
for c in aifb_rgat bgs_rgat mutag_rgat fb15k_rgcn aifb_hgt aifb_rgat_train bgs_rgat_train; do
  timeout 900 python bench.py --config $c --cuda-graph --no-ncu > gpurun_out/r02s/bench_${c}_graph.json 2>gpurun_out/r02s/bench_${c}_graph.err
  python -c "import json,sys; l=[x for x in open('gpurun_out/r02s/bench_${c}_graph.json') if x.startswith('{')][-1]; j=json.loads(l); print('$c graph', round(j['ms_per_step'],3), round(j['value']/1e9,3))"
done
timeout 900 python bench.py --impl reference > gpurun_out/r02s/bench_reference.json 2>&1; tail -c 400 gpurun_out/r02s/bench_reference.json; echo
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02s/launches_mag_hgt.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-ncu --no-e2e > /dev/null 2>&1; wc -l gpurun_out/r02s/launches_mag_hgt.csv
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_layers.py tests/test_gpu_segment_gemm.py tests/test_gpu_graph.py -q -x -k "not fullsize" > gpurun_out/r02s/memcheck.log 2>&1; echo "memcheck rc=$?"; tail -3 gpurun_out/r02s/memcheck.log
