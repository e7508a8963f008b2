# round 2: full GPU suite after the partition-aware node work + library-owned NCCL communicator
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02c_build.log 2>&1 || { tail -30 gpurun_out/r02c_build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02c_pytest.log 2>&1
tail -25 gpurun_out/r02c_pytest.log
timeout 600 python bench.py --no-cpu-baseline --no-ncu --comm --steps 10 > gpurun_out/r02c_bench_comm.log 2>&1; tail -1 gpurun_out/r02c_bench_comm.log | head -c 1500; echo
timeout 600 python bench.py --no-cpu-baseline --no-ncu --steps 10 > gpurun_out/r02c_bench.log 2>&1; tail -1 gpurun_out/r02c_bench.log | head -c 600; echo
