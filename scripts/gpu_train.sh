# F4: training-step parity tests + bench lines of the training configs
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_train.py tests/test_abi.py -q -x > gpurun_out/pytest_train.log 2>&1; tail -25 gpurun_out/pytest_train.log
for c in ${CONFIGS:-aifb_rgat_train am_rgat_train mag_hgt_train bgs_rgat_train}; do
  timeout 600 python bench.py --config $c --cpu-seconds 10 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -c 400 gpurun_out/bench_$c.err
done
