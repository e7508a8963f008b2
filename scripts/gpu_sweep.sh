# segment GEMM parity + d-sweep + ncu of the d=512 GEMM (tensor pipe), and the main tests
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_segment_gemm.py -q -x 2>&1 | tail -4
timeout 600 python scripts/gemm_sweep.py > gpurun_out/gemm_sweep.jsonl 2>gpurun_out/gemm_sweep.err
timeout 600 python scripts/gemm_sweep.py --no-gather --dims 512,1024 >> gpurun_out/gemm_sweep.jsonl 2>>gpurun_out/gemm_sweep.err
timeout 600 ncu --set full --clock-control none -k regex:k_gemm_ws -s 3 -c 1 -o gpurun_out/ncu_gemm512 python scripts/gemm_sweep.py --dims 512 --reps 1 > /dev/null 2>&1
timeout 1500 python -m pytest tests -q -x -m "gpu and not slow" 2>&1 | tail -4
python bench.py --config wikikg2_rgcn --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/bench_wikikg2_rgcn.json
