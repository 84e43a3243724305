mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/g_pytest.log 2>&1; tail -4 gpurun_out/g_pytest.log
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/g_bench_c4.json 2> gpurun_out/g_bench_c4.err; tail -1 gpurun_out/g_bench_c4.json
