# bench twice on one box (run-to-run variance) + RGAT/RGCN configs
python -c "import __graft_entry__ as g; g.build()"
python bench.py --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/benchA.json
python bench.py --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/benchB.json
