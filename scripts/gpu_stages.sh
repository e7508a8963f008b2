for S in 4 2 3; do
  RGNN_DEFINES="PAIR_BWD_STAGES=$S" python -m paper_2412_04747_b200.build > /dev/null 2>&1
  echo "== S=$S"
  timeout 300 python -m pytest tests/test_gpu_layers.py -q -x -k "bf16 and (tiny or aifb or am_shape)" 2>&1 | tail -1
  for c in mag_hgt wikikg2_rgcn mag_rgat; do
    timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('$c', round(d['ms_per_step'],3), round(k['pair_bwd_fused']['ms_per_step'],3))"
  done
done
