# k_gemm_tma with cp.async producer warps for gathered A: parity + A/B (RGNN_TMA=1 all / 2 contiguous only) + d-sweep
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02w_build.log 2>&1 || { tail -30 gpurun_out/r02w_build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_segment_gemm.py tests/test_gpu_layers.py -q -x > gpurun_out/r02w_pytest.log 2>&1; tail -2 gpurun_out/r02w_pytest.log
summ() { python - "$1" "$2" <<'PY'
import json, sys
ls=[x for x in open(sys.argv[1]) if x.startswith("{")]
if not ls: print(sys.argv[2], "no result"); sys.exit()
j=json.loads(ls[-1])
print(sys.argv[2], round(j["ms_per_step"],3), {k:round(v["ms_per_step"],3) for k,v in j["kernels"].items() if "gemm" in k})
PY
}
for c in mag_hgt am_rgat wikikg2_rgcn; do for v in 1 2; do RGNN_TMA=$v timeout 240 python bench.py --config $c --no-cpu-baseline --no-ncu --no-e2e --steps 20 > gpurun_out/r02w_${c}_$v.log 2>&1; summ gpurun_out/r02w_${c}_$v.log "$c TMA=$v"; done; done
timeout 600 python scripts/gemm_sweep.py > gpurun_out/r02w_sweep.jsonl 2>&1; cut -c1-150 gpurun_out/r02w_sweep.jsonl
