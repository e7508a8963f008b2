# smoke + GPU tests + bench of every config (1 GPU)
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -q -x -m "gpu and not slow" 2>&1 | tail -4
python bench.py --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_mag_hgt.json
for c in aifb_rgat am_rgat wikikg2_rgcn; do python bench.py --config $c --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/bench_$c.json; done
