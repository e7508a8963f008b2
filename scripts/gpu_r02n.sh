# TMA GEMM for contiguous A: D3 d-sweep (gathered: cp.async k_gemm_ws/tc; ungathered: TMA) + ncu tensor pipe at d=512
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02n_build.log 2>&1 || { tail -30 gpurun_out/r02n_build.log; exit 1; }
timeout 600 python scripts/gemm_sweep.py > gpurun_out/r02n_sweep.jsonl 2>&1; cut -c1-200 gpurun_out/r02n_sweep.jsonl
timeout 600 python scripts/gemm_sweep.py --no-gather > gpurun_out/r02n_sweep_ng.jsonl 2>&1; cut -c1-200 gpurun_out/r02n_sweep_ng.jsonl
RGNN_TMA=0 timeout 600 python scripts/gemm_sweep.py --no-gather > gpurun_out/r02n_sweep_ng_tma0.jsonl 2>&1; cut -c1-200 gpurun_out/r02n_sweep_ng_tma0.jsonl
timeout 600 ncu --set full --clock-control none -k regex:"k_gemm" -c 2 -o gpurun_out/r02n_ncu_d512 python scripts/gemm_sweep.py --no-gather --dims 512 --reps 1 > gpurun_out/r02n_ncu.log 2>&1; tail -1 gpurun_out/r02n_ncu.log
timeout 600 ncu --set full --clock-control none -k regex:"k_gemm" -c 2 -o gpurun_out/r02n_ncu_d512g python scripts/gemm_sweep.py --dims 512 --reps 1 > gpurun_out/r02n_ncug.log 2>&1; tail -1 gpurun_out/r02n_ncug.log
