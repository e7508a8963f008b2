# round-1 closing check: smoke, the whole GPU suite, default bench line
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
mkdir -p gpurun_out/fin3
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -2 > gpurun_out/fin3/pytest_gpu.txt; cat gpurun_out/fin3/pytest_gpu.txt
python bench.py 2>&1 | tail -1 > gpurun_out/fin3/bench_mag_hgt.json
python bench.py --config mag_hgt_train --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/fin3/bench_mag_hgt_train.json
python bench.py --config am_rgat_train --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/fin3/bench_am_rgat_train.json
python bench.py --impl reference --steps 3 --warmup 3 2>&1 | tail -1 > gpurun_out/fin3/bench_reference.json
