# F4 train configs (+ CUDA graph on the small ones), D1 a_dst sensitivity, extra shapes, GPU tests
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -q -x -m "gpu and not slow" > gpurun_out/pytest_gpu2.log 2>&1; tail -3 gpurun_out/pytest_gpu2.log
run() { n=$1; shift; timeout 600 python bench.py "$@" > gpurun_out/b2_$n.json 2> gpurun_out/b2_$n.err; tail -c 300 gpurun_out/b2_$n.err; }
run mag_hgt --cpu-seconds 10
run aifb_rgat_train_graph --config aifb_rgat_train --cuda-graph --no-cpu-baseline
run bgs_rgat_train_graph --config bgs_rgat_train --cuda-graph --no-cpu-baseline
run am_rgat_train --config am_rgat_train --cpu-seconds 10
run mag_hgt_train --config mag_hgt_train --no-cpu-baseline
run mag_hgt_adst0 --a-dst 0 --no-cpu-baseline --no-e2e
run mag_hgt_adst12 --a-dst 1.2 --no-cpu-baseline --no-e2e
run mutag_rgat --config mutag_rgat --no-cpu-baseline --cuda-graph
run fb15k_rgcn --config fb15k_rgcn --no-cpu-baseline --cuda-graph
run biokg_hgt --config biokg_hgt --no-cpu-baseline
