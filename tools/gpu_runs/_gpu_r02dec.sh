for sp in 8 10 12; do python tools/phase_trace.py $sp 64 300 2>&1 | head -6 | tail -5 | sed "s/^/S=$sp /"; done
for c in 1 2; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c$c', d['value'], d['roofline']['frac'], d['e2e']['value'])"; done
timeout 900 python -m pytest tests/test_device_parity.py tests/test_error_contract.py -m gpu -x -q 2>&1 | tail -2
