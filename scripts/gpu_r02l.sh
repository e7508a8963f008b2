# full GPU suite + smoke + default bench after the pair-pass cleanup (split-halves bf16 group kernel)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02l_build.log 2>&1 || { tail -30 gpurun_out/r02l_build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02l_pytest.log 2>&1; tail -4 gpurun_out/r02l_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02l_smoke.log 2>&1; tail -2 gpurun_out/r02l_smoke.log
timeout 900 python bench.py > gpurun_out/r02l_bench.log 2>&1; tail -1 gpurun_out/r02l_bench.log | head -c 1500; echo
