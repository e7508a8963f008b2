# bwd_pair occupancy sweep beyond 4 blocks/SM (rebuilds librgnn.so on the box for each variant)
for v in "UNR_P=2 PAIR_MINB=4" "UNR_P=2 PAIR_MINB=5" "UNR_P=2 PAIR_MINB=6" "UNR_P=1 PAIR_MINB=6" "UNR_P=1 PAIR_MINB=8"; do
  RGNN_DEFINES="$v" python -m paper_2412_04747_b200.build > /dev/null 2>&1
  echo "== $v"
  python bench.py --no-cpu-baseline --no-e2e --steps 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print(round(d['ms_per_step'],3), {n: round(v['ms_per_step'],3) for n,v in k.items() if 'pair' in n})"
done
