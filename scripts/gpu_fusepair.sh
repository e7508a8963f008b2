python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_layers.py -q -x -k "bf16 or tiny" 2>&1 | tail -2
q() { timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print(round(d['ms_per_step'],3), {n: round(v['ms_per_step'],3) for n,v in k.items() if 'gemm' in n or 'wgrad' in n or 'fused' in n or 'seg' in n})"; }
for c in mag_hgt wikikg2_rgcn mag_rgat am_hgt; do echo "== $c fuse=0"; RGNN_FUSE_PAIR=0 q --config $c; echo "== $c fuse=1"; q --config $c; done
