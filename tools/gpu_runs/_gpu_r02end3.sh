# final code: smoke, full GPU suite, headline bench (driver form), config 3 and its 512-replica split
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/end3_smoke.log 2>&1; tail -1 gpurun_out/end3_smoke.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/end3_gputests.log 2>&1; tail -1 gpurun_out/end3_gputests.log
timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/end3_bench_config4.json 2>/dev/null
timeout 900 python bench.py --config 3 --replicas 512 --steps 3 > gpurun_out/end3_bench_config3_r512.json 2>/dev/null
for f in end3_bench_config4 end3_bench_config3_r512; do tail -1 gpurun_out/$f.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', d['value'], d['roofline']['frac'], d['e2e']['value'], d['gpu_launches'], d['clocks']['sm_mhz'], d['clocks']['reasons'], (d.get('cpu_baseline') or {}).get('value'))"; done
