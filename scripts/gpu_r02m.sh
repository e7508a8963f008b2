# TMA GEMM generation (k_gemm_tma): GEMM parity, layer parity, A/B bench, d-sweep, SASS check
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02m_build.log 2>&1 || { tail -30 gpurun_out/r02m_build.log; exit 1; }
cuobjdump -sass paper_2412_04747_b200/librgnn.so | grep -c UTMALDG > gpurun_out/r02m_sass_utmaldg.txt
timeout 900 python -m pytest tests/test_gpu_segment_gemm.py -q -x > gpurun_out/r02m_pytest_gemm.log 2>&1; tail -3 gpurun_out/r02m_pytest_gemm.log
timeout 900 python -m pytest tests/test_gpu_layers.py -q -x > gpurun_out/r02m_pytest_layers.log 2>&1; tail -3 gpurun_out/r02m_pytest_layers.log
summ() { python - "$1" "$2" <<'PY'
import json, sys
l=[x for x in open(sys.argv[1]) if x.startswith("{")][-1]; j=json.loads(l)
print(sys.argv[2], round(j["ms_per_step"],3), {k:round(v["ms_per_step"],3) for k,v in j["kernels"].items() if "gemm" in k or "wgrad" in k or "fused" in k})
PY
}
for v in 1 0; do RGNN_TMA=$v timeout 600 python bench.py --no-cpu-baseline --no-ncu --no-e2e --steps 20 > gpurun_out/r02m_tma$v.log 2>&1; summ gpurun_out/r02m_tma$v.log "TMA=$v"; done
RGNN_TMA=1 timeout 600 python scripts/gemm_sweep.py > gpurun_out/r02m_sweep_tma.jsonl 2>&1; cat gpurun_out/r02m_sweep_tma.jsonl | cut -c1-300
RGNN_TMA=1 timeout 600 python scripts/gemm_sweep.py --no-gather > gpurun_out/r02m_sweep_tma_ng.jsonl 2>&1; cat gpurun_out/r02m_sweep_tma_ng.jsonl | cut -c1-300
