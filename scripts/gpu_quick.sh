# quick loop: build, the layer parity tests for $K (pytest -k), and bench lines for $CONFIGS
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_layers.py tests/test_gpu_fullsize.py -q -x -k "${K:-hgt}" 2>&1 | tail -2
for c in ${CONFIGS:-mag_hgt}; do
  python bench.py --config $c --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/q_$c.json
done
