python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_layers.py -q -x -k "rgat or rgcn" 2>&1 | tail -2
q() { python bench.py --no-cpu-baseline --no-e2e --steps 10 "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print(round(d['ms_per_step'],3), {n: round(v['ms_per_step'],3) for n,v in k.items() if 'pair' in n})"; }
for c in am_rgat mag_rgat; do echo "== $c stage=0"; RGNN_STAGE=0 q --config $c; echo "== $c stage=1"; q --config $c; done
for u in 1 2 4; do RGNN_DEFINES="UNR_R=$u" python -m paper_2412_04747_b200.build > /dev/null 2>&1; echo "== wikikg2 UNR_R=$u"; q --config wikikg2_rgcn; done
