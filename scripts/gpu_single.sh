python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests -q -x -m gpu 2>&1 | tail -2
q() { timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print(round(d['ms_per_step'],3), {n: round(v['ms_per_step'],3) for n,v in k.items() if ('pair' in n or 'dst' in n) and v['ms_per_step'] > 0.03})"; }
for c in mag_hgt am_rgat am_hgt mag_rgat; do echo "== $c single=0"; RGNN_SINGLE=0 q --config $c; echo "== $c single=1"; q --config $c; done
echo "== am_rgat vanilla single=0"; RGNN_SINGLE=0 q --config am_rgat --no-compact; echo "== am_rgat vanilla single=1"; q --config am_rgat --no-compact
