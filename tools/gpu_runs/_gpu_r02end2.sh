# after the staged gate pass: full GPU suite, smoke, config 3 / 4 / 5 bench lines
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/end2_smoke.log 2>&1; tail -1 gpurun_out/end2_smoke.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/end2_gputests.log 2>&1; tail -1 gpurun_out/end2_gputests.log
timeout 900 python bench.py --config 3 --steps 2 > gpurun_out/end2_bench_config3.json 2>/dev/null
timeout 900 python bench.py --config 3 --replicas 512 --steps 3 > gpurun_out/end2_bench_config3_r512.json 2>/dev/null
timeout 900 python bench.py > gpurun_out/end2_bench_config4.json 2>/dev/null
for f in end2_bench_config3 end2_bench_config3_r512 end2_bench_config4; do tail -1 gpurun_out/$f.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', d['value'], d['roofline']['frac'], d['roofline'].get('kernel'), d['e2e']['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/r02_traffic_config3_end.csv python bench.py --config 3 --mc-steps 100 --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1; wc -l gpurun_out/r02_traffic_config3_end.csv
