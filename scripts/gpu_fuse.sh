python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_layers.py tests/test_gpu_fullsize.py -q -x -k "hgt" 2>&1 | tail -1
q() { python bench.py --no-cpu-baseline --no-e2e --steps 10 "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print(round(d['ms_per_step'],3), {n: round(v['ms_per_step'],3) for n,v in k.items() if 'gemm' in n or 'seg' in n})"; }
for c in mag_hgt am_hgt; do echo "== $c fuse=0"; RGNN_FUSE_RED=0 q --config $c; echo "== $c fuse=1"; RGNN_FUSE_RED=1 q --config $c; done
