python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -q -x -m "gpu and not slow" 2>&1 | tail -4
for c in mag_hgt am_rgat wikikg2_rgcn; do
  python bench.py --config $c --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/bench_ws_$c.json
  RGNN_GEMM_WS=0 python bench.py --config $c --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/bench_nows_$c.json
done
