# staged gate with a producer warp (no CTA barrier per chunk)
mkdir -p gpurun_out
python tools/phase_trace.py 16 148 20 2>&1 | head -3 | tail -2
timeout 600 python bench.py --config 3 --mc-steps 200 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 4096x200', d['value'], d['roofline']['frac'])"
timeout 600 python bench.py --config 3 --replicas 512 --mc-steps 300 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 512x300', d['value'], d['roofline']['frac'])"
timeout 900 python -m pytest tests/test_device_parity.py tests/test_queue_schedule.py tests/test_fuzz_parity.py -m gpu -q -x > gpurun_out/gprod_t.log 2>&1; tail -1 gpurun_out/gprod_t.log; grep FAILED gpurun_out/gprod_t.log | head -3
