# RGAT weighted-SpMM pair pass (RGNN_RGATW): parity (all RGAT tests) + A/B on am_rgat / mag_rgat
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02r_build.log 2>&1 || { tail -30 gpurun_out/r02r_build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -x -k "rgat" > gpurun_out/r02r_pytest.log 2>&1; tail -3 gpurun_out/r02r_pytest.log
summ() { python - "$1" "$2" <<'PY'
import json, sys
l=[x for x in open(sys.argv[1]) if x.startswith("{")][-1]; j=json.loads(l)
print(sys.argv[2], round(j["ms_per_step"],3), {k:round(v["ms_per_step"],3) for k,v in j["kernels"].items() if v["ms_per_step"]>0.02})
PY
}
for c in am_rgat mag_rgat; do for v in 1 0; do RGNN_RGATW=$v timeout 600 python bench.py --config $c --no-cpu-baseline --no-ncu --no-e2e --steps 20 > gpurun_out/r02r_${c}_$v.log 2>&1; summ gpurun_out/r02r_${c}_$v.log "$c RGATW=$v"; done; done
