# staged gate on 2- and 4-CTA clusters (512 replicas of L=16: the model picks CS = 2)
for v in 0 1; do
  TG_GATE_BULK=$v timeout 600 python bench.py --config 3 --replicas 512 --mc-steps 300 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 512x300 knob $v', d['value'], d['roofline']['frac'])"
  TG_GATE_BULK=$v timeout 600 python bench.py --config 3 --replicas 32 --mc-steps 300 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 32x300 (CS=4) knob $v', d['value'], d['roofline']['frac'])"
done
timeout 900 python -m pytest tests/test_device_parity.py tests/test_queue_schedule.py tests/test_fuzz_parity.py -m gpu -q > gpurun_out/gbulk_cs_t.log 2>&1; tail -1 gpurun_out/gbulk_cs_t.log; grep FAILED gpurun_out/gbulk_cs_t.log | head
