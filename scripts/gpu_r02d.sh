# round 2 re-entry: full GPU suite + smoke + default bench + comm bench on the committed HEAD
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02d_build.log 2>&1 || { tail -30 gpurun_out/r02d_build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02d_pytest.log 2>&1
tail -25 gpurun_out/r02d_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02d_smoke.log 2>&1; tail -3 gpurun_out/r02d_smoke.log
timeout 900 python bench.py > gpurun_out/r02d_bench.log 2>&1; tail -1 gpurun_out/r02d_bench.log | head -c 4000; echo
timeout 600 python bench.py --no-cpu-baseline --no-ncu --comm --steps 10 > gpurun_out/r02d_bench_comm.log 2>&1; tail -1 gpurun_out/r02d_bench_comm.log | head -c 1500; echo
