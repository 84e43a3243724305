# TMA-staged gate pass for S >= 16 (cluster schedule): A/B (TG_GATE_BULK), parity tests
mkdir -p gpurun_out
for v in 0 1; do
  echo "== TG_GATE_BULK=$v"
  TG_GATE_BULK=$v python tools/phase_trace.py 16 148 20 2>&1 | head -4 | tail -3
  TG_GATE_BULK=$v timeout 600 python bench.py --config 3 --mc-steps 200 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 4096x200', d['value'], d['roofline']['frac'], d['config'].get('schedule', d['roofline'].get('kernel')))"
done
timeout 900 python -m pytest tests/test_device_parity.py tests/test_queue_schedule.py tests/test_fuzz_parity.py -m gpu -q -x > gpurun_out/gbulk_t.log 2>&1; tail -1 gpurun_out/gbulk_t.log; grep -E "FAILED|Error" gpurun_out/gbulk_t.log | head -5
