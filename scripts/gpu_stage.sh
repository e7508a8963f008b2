# staged (smem K~/M) group-mode HGT pair kernel vs the register-resident one; U sweep
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_layers.py -q -x -k hgt 2>&1 | tail -2
q() { python bench.py --no-cpu-baseline --no-e2e --steps 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print(round(d['ms_per_step'],3), {n: round(v['ms_per_step'],3) for n,v in k.items() if 'pair' in n})"; }
echo "== register (RGNN_STAGE=0)"; RGNN_STAGE=0 q
for u in 3 2 4; do
  RGNN_DEFINES="UNR_S=$u" python -m paper_2412_04747_b200.build > /dev/null 2>&1
  echo "== staged U=$u"; q
done
