python tools/phase_trace.py 12 148 300 2>&1 | head -6 | tail -5
for i in 1 2; do timeout 300 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2', d['value'], d['roofline']['frac'], d['e2e']['value'])"; done
timeout 900 python -m pytest tests/test_device_parity.py tests/test_error_contract.py tests/test_cli.py tests/test_integration_reference_api.py -m gpu -q > gpurun_out/defer_t.log 2>&1; tail -1 gpurun_out/defer_t.log; grep FAILED gpurun_out/defer_t.log | head
