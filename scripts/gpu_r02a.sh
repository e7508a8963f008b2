set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02a_build.log 2>&1
nvidia-smi > gpurun_out/r02a_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02a_pytest.log 2>&1
tail -3 gpurun_out/r02a_pytest.log
python bench.py > gpurun_out/r02a_bench.log 2>&1; tail -1 gpurun_out/r02a_bench.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02a_smoke.log 2>&1; tail -2 gpurun_out/r02a_smoke.log
