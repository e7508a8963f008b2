# round 2: parity additions (full-size shapes, degenerate pow2 graph, sym partition, wide fp32 rows,
# binding checks, F4 flat tolerance) + bench with the new roofline accounting and in-run ncu traffic
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02b_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -k "fullsize or degenerate or partition or wide_rows or bad_shapes or two_layer or wikikg2" > gpurun_out/r02b_pytest.log 2>&1
tail -15 gpurun_out/r02b_pytest.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r02b_bench.log 2>&1; tail -1 gpurun_out/r02b_bench.log | head -c 3000
