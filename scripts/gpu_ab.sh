# A/B: HEAD build (ab_head/) vs working tree, same box, same flags.  usage: gpu_ab.sh TAG [extra bench args]
tag=$1; shift
summ() { python - "$1" "$2" <<'PY'
import json, sys
l=[x for x in open(sys.argv[1]) if x.startswith("{")][-1]; j=json.loads(l)
print(sys.argv[2], round(j["ms_per_step"],3), {k:round(v["ms_per_step"],3) for k,v in j["kernels"].items() if v["ms_per_step"] > 0.05})
PY
}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1 || { tail -30 gpurun_out/${tag}_build.log; exit 1; }
(cd ab_head && python -c "import __graft_entry__ as g; g.build()" > ../gpurun_out/${tag}_build_head.log 2>&1)
for i in 1 2; do
(cd ab_head && timeout 600 python bench.py --no-cpu-baseline --no-ncu --no-e2e --steps 20 "$@" > ../gpurun_out/${tag}_head$i.log 2>&1); summ gpurun_out/${tag}_head$i.log HEAD
for w in 0 1; do RGNN_PAIRW=$w timeout 600 python bench.py --no-cpu-baseline --no-ncu --no-e2e --steps 20 "$@" > gpurun_out/${tag}_w$w.$i.log 2>&1; summ gpurun_out/${tag}_w$w.$i.log "NEW PAIRW=$w"; done
done
