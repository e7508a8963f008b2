python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_layers.py tests/test_gpu_train.py -q -x -k "hgt" 2>&1 | tail -2
q() { python bench.py --no-cpu-baseline --no-e2e --steps 10 "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print(round(d['ms_per_step'],3), {n: round(v['ms_per_step'],3) for n,v in k.items() if v['ms_per_step'] > 0.08})"; }
for c in mag_hgt am_hgt; do echo "== $c overlap=0"; RGNN_OVERLAP=0 q --config $c; echo "== $c overlap=1"; q --config $c; done
