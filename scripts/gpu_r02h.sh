# bulk-copy ring pair pass: parity (HGT) + A/B vs the work-plan kernels + ncu
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02h_build.log 2>&1 || { tail -30 gpurun_out/r02h_build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x -k "hgt" > gpurun_out/r02h_pytest.log 2>&1; tail -3 gpurun_out/r02h_pytest.log
summ() { python - "$1" "$2" <<'PY'
import json, sys
l=[x for x in open(sys.argv[1]) if x.startswith("{")][-1]; j=json.loads(l)
print(sys.argv[2], round(j["ms_per_step"],3), {k:round(v["ms_per_step"],3) for k,v in j["kernels"].items() if v["ms_per_step"] > 0.05})
PY
}
for b in 1 0; do RGNN_BULK=$b timeout 600 python bench.py --no-cpu-baseline --no-ncu --no-e2e --steps 20 > gpurun_out/r02h_b$b.log 2>&1; summ gpurun_out/r02h_b$b.log "BULK=$b"; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_hgt_bwd_pair_bulk" -c 1 -o gpurun_out/r02h_bulk python bench.py --no-cpu-baseline --no-ncu --no-e2e --steps 1 --warmup 1 > gpurun_out/r02h_ncu.log 2>&1; tail -2 gpurun_out/r02h_ncu.log
