# RGAT baselines: am_rgat / mag_rgat per-kernel breakdown + ncu of the RGAT traversal kernels (AM)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02o_build.log 2>&1 || { tail -30 gpurun_out/r02o_build.log; exit 1; }
summ() { python - "$1" "$2" <<'PY'
import json, sys
l=[x for x in open(sys.argv[1]) if x.startswith("{")][-1]; j=json.loads(l)
print(sys.argv[2], round(j["ms_per_step"],3), j["config"].get("pairs"), {k:round(v["ms_per_step"],3) for k,v in j["kernels"].items() if v["ms_per_step"]>0.02})
PY
}
for c in am_rgat mag_rgat; do timeout 600 python bench.py --config $c --no-cpu-baseline --no-ncu --no-e2e --steps 20 > gpurun_out/r02o_$c.log 2>&1; summ gpurun_out/r02o_$c.log $c; done
timeout 900 ncu --set full --clock-control none -k regex:"k_rgat" -o gpurun_out/r02o_ncu_am python bench.py --config am_rgat --no-cpu-baseline --no-ncu --no-e2e --steps 1 --warmup 1 > gpurun_out/r02o_ncu.log 2>&1; tail -1 gpurun_out/r02o_ncu.log
