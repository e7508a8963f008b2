# warp-specialized TMA fused pair backward (k_pair_bwd_ws): parity + A/B on mag_hgt, wikikg2_rgcn, am_rgat
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02v_build.log 2>&1 || { tail -30 gpurun_out/r02v_build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_layers.py tests/test_gpu_train.py tests/test_gpu_partition.py -q -x > gpurun_out/r02v_pytest.log 2>&1; tail -3 gpurun_out/r02v_pytest.log
summ() { python - "$1" "$2" <<'PY'
import json, sys
l=[x for x in open(sys.argv[1]) if x.startswith("{")][-1]; j=json.loads(l)
print(sys.argv[2], round(j["ms_per_step"],3), {k:round(v["ms_per_step"],3) for k,v in j["kernels"].items() if "fused" in k or "wgrad_reduce" in k})
PY
}
for c in mag_hgt wikikg2_rgcn am_rgat; do for v in 1 0; do RGNN_PAIR_WS=$v timeout 240 python bench.py --config $c --no-cpu-baseline --no-ncu --no-e2e --steps 20 > gpurun_out/r02v_${c}_$v.log 2>&1; summ gpurun_out/r02v_${c}_$v.log "$c WS=$v"; done; done
