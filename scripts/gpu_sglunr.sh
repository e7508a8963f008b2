q() { timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 "$@" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print(round(d['ms_per_step'],3), {n: round(v['ms_per_step'],3) for n,v in k.items() if n in ('rgat_bwd_dst','rgat_bwd_pair')})"; }
for u in 4 2 3 1; do
  RGNN_DEFINES="UNR_SGL=$u" python -m paper_2412_04747_b200.build > /dev/null 2>&1
  echo "== UNR_SGL=$u"; q --config am_rgat
done
timeout 600 python -m pytest tests/test_gpu_layers.py -q -k "rgat and (am_shape or degenerate or tiny)" 2>&1 | tail -1
