# weighted pair SpMM (k_pair_spmm) vs the recomputing pair kernels on HGT; parity + bench + ncu
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02e_build.log 2>&1 || { tail -30 gpurun_out/r02e_build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x -k "hgt" > gpurun_out/r02e_pytest.log 2>&1; tail -5 gpurun_out/r02e_pytest.log
for w in 1 0; do
RGNN_PAIRW=$w timeout 600 python bench.py --no-cpu-baseline --no-ncu --no-e2e --steps 20 > gpurun_out/r02e_bench_w$w.log 2>&1
python - <<PY
import json
l=[x for x in open("gpurun_out/r02e_bench_w$w.log") if x.startswith("{")][-1]; j=json.loads(l)
print("PAIRW=$w", round(j["ms_per_step"],3), {k:round(v["ms_per_step"],3) for k,v in j["kernels"].items() if "hgt" in k or "pair" in k})
PY
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pair_spmm -c 1 -o gpurun_out/r02e_spmm python bench.py --no-cpu-baseline --no-ncu --no-e2e --steps 1 --warmup 1 > gpurun_out/r02e_ncu.log 2>&1; tail -3 gpurun_out/r02e_ncu.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_hgt|k_pair|k_merge" --csv python bench.py --no-cpu-baseline --no-ncu --no-e2e --steps 1 --warmup 1 > gpurun_out/r02e_ncu_list.csv 2>&1; tail -3 gpurun_out/r02e_ncu_list.csv
