q() { python bench.py --no-cpu-baseline --no-e2e --steps 10 "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print(round(d['ms_per_step'],3), {n: round(v['ms_per_step'],3) for n,v in k.items() if 'trav' in n or 'dst' in n})"; }
for v in ${VARIANTS}; do
  RGNN_DEFINES="$(echo $v | tr , " ")" python -m paper_2412_04747_b200.build > /dev/null 2>&1
  echo "== $v"; q $ARGS
done
