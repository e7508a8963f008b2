# seg_reduce_rows with the row-index list prefetched a batch ahead: parity + wikikg2 / am_rgat timing
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02x_build.log 2>&1 || { tail -30 gpurun_out/r02x_build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_layers.py -q -x -k "rgcn or rgat" > gpurun_out/r02x_pytest.log 2>&1; tail -2 gpurun_out/r02x_pytest.log
for c in wikikg2_rgcn am_rgat; do timeout 240 python bench.py --config $c --no-cpu-baseline --no-ncu --no-e2e --steps 20 > gpurun_out/r02x_${c}.log 2>&1; python - gpurun_out/r02x_${c}.log $c <<'PY'
import json, sys
j=json.loads([x for x in open(sys.argv[1]) if x.startswith("{")][-1])
print(sys.argv[2], round(j["ms_per_step"],3), {k:round(v["ms_per_step"],3) for k,v in j["kernels"].items() if "reduce" in k})
PY
done
