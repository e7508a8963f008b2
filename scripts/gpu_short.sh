# short-item kernels (KI items per lane group) vs the plain group mode
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_layers.py tests/test_gpu_fullsize.py -q -x -k "${K:-hgt or rgcn}" 2>&1 | tail -2
q() { python bench.py --no-cpu-baseline --no-e2e --steps 10 "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print(round(d['ms_per_step'],3), {n: round(v['ms_per_step'],3) for n,v in k.items() if 'pair' in n or 'trav' in n or 'dst' in n})"; }
for c in ${CONFIGS:-mag_hgt am_hgt}; do
  echo "== $c short=0"; RGNN_SHORT=0 q --config $c
  echo "== $c short=1"; q --config $c
done
