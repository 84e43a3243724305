# End-of-round evidence: smoke, the full GPU suite, and one bench line per config (profiles/r02_end_*).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/end_smoke.log 2>&1; tail -1 gpurun_out/end_smoke.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/end_gputests.log 2>&1; tail -1 gpurun_out/end_gputests.log
timeout 900 python bench.py > gpurun_out/end_bench_config4.json 2> gpurun_out/end_bench_config4.err
timeout 600 python bench.py --config 1 > gpurun_out/end_bench_config1.json 2>/dev/null
timeout 600 python bench.py --config 2 > gpurun_out/end_bench_config2.json 2>/dev/null
timeout 900 python bench.py --config 3 --steps 2 > gpurun_out/end_bench_config3.json 2>/dev/null
timeout 600 python bench.py --config 5 > gpurun_out/end_bench_config5.json 2>/dev/null
for c in 1 2 3 4 5; do tail -1 gpurun_out/end_bench_config$c.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c$c', d['value'], d['roofline']['frac'], d['e2e']['value'], d['gpu_launches'], d['clocks']['sm_mhz'], d['clocks']['reasons'], (d.get('cpu_baseline') or {}).get('value'))"; done
