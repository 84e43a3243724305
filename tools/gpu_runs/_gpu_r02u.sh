timeout 1200 python -m pytest tests/test_queue_schedule.py -x -q 2>&1 | tail -2
mkdir -p gpurun_out; timeout 1200 compute-sanitizer --tool racecheck --print-limit 30 python tools/sanitizer_run.py > gpurun_out/race2.txt 2>&1; tail -2 gpurun_out/race2.txt
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4', d['value'], round(d['roofline']['frac'],4), d['roofline']['kernel'])"
