# TMA-staged gate: decomposition (bit 0 staged gate, bit 1 start offsets) and S = 14 / 15
for v in 0 1 2 3; do
  TG_GATE_BULK=$v timeout 600 python bench.py --config 3 --mc-steps 200 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 4096x200 knob $v', d['value'], d['roofline']['frac'])"
done
for v in 0 1 3; do
  TG_GATE_BULK_MIN=13 TG_GATE_BULK=$v timeout 600 python bench.py --config 5 --replicas 16384 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 16384x100 knob $v', d['value'], d['roofline']['frac'])"
  TG_GATE_BULK_MIN=13 TG_GATE_BULK=$v python tools/phase_trace.py 14 148 30 2>&1 | head -3 | tail -2
done
TG_GATE_BULK_MIN=13 timeout 900 python -m pytest tests/test_device_parity.py -m gpu -q -x -k "14 or 13 or hbm or cluster" > gpurun_out/gbulk2_t.log 2>&1; tail -1 gpurun_out/gbulk2_t.log; grep FAILED gpurun_out/gbulk2_t.log | head -3
