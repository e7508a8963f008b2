# bf16 HGT pair pass with 4 columns per lane at full occupancy: parity + A/B
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02j_build.log 2>&1 || { tail -30 gpurun_out/r02j_build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x -k "hgt" > gpurun_out/r02j_pytest.log 2>&1; tail -2 gpurun_out/r02j_pytest.log
summ() { python - "$1" "$2" <<'PY'
import json, sys
l=[x for x in open(sys.argv[1]) if x.startswith("{")][-1]; j=json.loads(l)
print(sys.argv[2], round(j["ms_per_step"],3), {k:round(v["ms_per_step"],3) for k,v in j["kernels"].items() if "pair" in k})
PY
}
for v in "RGNN_HALF=0" "RGNN_PAIRH_MINB=8" "RGNN_PAIRH_MINB=7" "RGNN_PAIRH_MINB=6" "RGNN_SHORT=0"; do env $v timeout 600 python bench.py --no-cpu-baseline --no-ncu --no-e2e --steps 20 > gpurun_out/r02j_$v.log 2>&1; summ gpurun_out/r02j_$v.log "$v"; done
timeout 900 ncu --set full --clock-control none -k regex:"k_hgt_bwd_pair" -c 3 -o gpurun_out/r02j_ncu python bench.py --no-cpu-baseline --no-ncu --no-e2e --steps 1 --warmup 1 > gpurun_out/r02j_ncu.log 2>&1; tail -1 gpurun_out/r02j_ncu.log
