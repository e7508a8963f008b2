# pair pass A/B: recompute (PAIRW=0) vs weighted SpMM (PAIRW=1) after the WT template split
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02f_build.log 2>&1 || { tail -30 gpurun_out/r02f_build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x -k "hgt" > gpurun_out/r02f_pytest.log 2>&1; tail -3 gpurun_out/r02f_pytest.log
for w in 1 0; do
RGNN_PAIRW=$w timeout 600 python bench.py --no-cpu-baseline --no-ncu --no-e2e --steps 20 > gpurun_out/r02f_bench_w$w.log 2>&1
python - <<PY
import json
l=[x for x in open("gpurun_out/r02f_bench_w$w.log") if x.startswith("{")][-1]; j=json.loads(l)
print("PAIRW=$w", round(j["ms_per_step"],3), {k:round(v["ms_per_step"],3) for k,v in j["kernels"].items() if "hgt" in k or "pair" in k})
PY
done
timeout 900 ncu --set full --clock-control none -k regex:"k_pair_spmm|k_hgt_bwd_dst" -c 4 -o gpurun_out/r02f_ncu python bench.py --no-cpu-baseline --no-ncu --no-e2e --steps 1 --warmup 1 > gpurun_out/r02f_ncu.log 2>&1; tail -2 gpurun_out/r02f_ncu.log
