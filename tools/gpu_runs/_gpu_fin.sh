mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/fin_c2.json 2> /dev/null
timeout 300 python bench.py --config 1 --no-cpu-baseline > gpurun_out/fin_c1.json 2> /dev/null
for c in 3 4; do timeout 400 python bench.py --config $c --steps 2 --no-cpu-baseline > gpurun_out/fin_c$c.json 2> /dev/null; done
timeout 300 python bench.py --config 5 --no-cpu-baseline > gpurun_out/fin_c5.json 2> /dev/null
for c in 1 2 3 4 5; do tail -1 gpurun_out/fin_c$c.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c$c', d['value'], d['roofline']['frac'], d['e2e']['value'], d['gpu_launches'], d['clocks']['reasons'], (d.get('cpu_baseline') or {}).get('value'))"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin_launches_c5.csv python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; wc -l gpurun_out/fin_launches_c5.csv
