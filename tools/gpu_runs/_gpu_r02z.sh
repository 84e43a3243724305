mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/z_smoke.log 2>&1; tail -2 gpurun_out/z_smoke.log
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/z_gputests.log 2>&1; tail -3 gpurun_out/z_gputests.log
timeout 900 python bench.py > gpurun_out/z_bench.json 2> gpurun_out/z_bench.err; tail -1 gpurun_out/z_bench.json
