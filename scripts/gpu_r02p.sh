# fp32 GEMM / wgrad kernels (FFMA2, register-tiled): parity + mag_hgt_f32 A/B; ncu of the AM RGAT traversal
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02p_build.log 2>&1 || { tail -30 gpurun_out/r02p_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_segment_gemm.py tests/test_gpu_layers.py -q -x -k "f32 or fp32 or float" > gpurun_out/r02p_pytest.log 2>&1; tail -3 gpurun_out/r02p_pytest.log
summ() { python - "$1" "$2" <<'PY'
import json, sys
l=[x for x in open(sys.argv[1]) if x.startswith("{")][-1]; j=json.loads(l)
print(sys.argv[2], round(j["ms_per_step"],3), {k:round(v["ms_per_step"],3) for k,v in j["kernels"].items() if v["ms_per_step"]>0.05})
PY
}
for v in 1 0; do RGNN_F32GEMM=$v timeout 600 python bench.py --config mag_hgt_f32 --no-cpu-baseline --no-ncu --no-e2e --steps 10 > gpurun_out/r02p_f32_$v.log 2>&1; summ gpurun_out/r02p_f32_$v.log "F32GEMM=$v"; done
timeout 900 ncu --set full --clock-control none -k regex:"k_rgat_bwd_dst|k_rgat_fwd|k_rgat_bwd_pair" -c 6 -o gpurun_out/r02p_ncu_am_rgat python bench.py --config am_rgat --no-cpu-baseline --no-ncu --no-e2e --steps 1 --warmup 1 > gpurun_out/r02p_ncu.log 2>&1; tail -1 gpurun_out/r02p_ncu.log
