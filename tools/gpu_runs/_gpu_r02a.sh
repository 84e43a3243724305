set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/a_smoke.log 2>&1; tail -3 gpurun_out/a_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/a_pytest.log 2>&1; tail -15 gpurun_out/a_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/a_bench_c4.json 2> gpurun_out/a_bench_c4.err; tail -1 gpurun_out/a_bench_c4.json; tail -5 gpurun_out/a_bench_c4.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/a_ref_c4.json 2> gpurun_out/a_ref_c4.err; tail -1 gpurun_out/a_ref_c4.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/a_launches_c4.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; wc -l gpurun_out/a_launches_c4.csv
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active --clock-control none -k regex:anneal_hbm -c 1 --csv --log-file gpurun_out/a_traffic_c4.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; tail -5 gpurun_out/a_traffic_c4.csv
