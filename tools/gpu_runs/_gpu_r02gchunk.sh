# staged gate: chunk size / ring depth sweep at S = 16 and S = 14
mkdir -p gpurun_out
for c in 1024 512 256; do
  TG_GATE_CHUNK=$c timeout 600 python bench.py --config 3 --mc-steps 200 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 4096x200 chunk $c', d['value'], d['roofline']['frac'])"
  TG_GATE_CHUNK=$c python tools/phase_trace.py 16 148 20 2>&1 | head -3 | tail -1
done
TG_GATE_BULK=0 timeout 600 python bench.py --config 5 --replicas 16384 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 16384 register path', d['value'], d['roofline']['frac'])"
TG_GATE_BULK=0 python tools/phase_trace.py 14 148 30 2>&1 | head -3 | tail -1
for c in 512 256 128; do
  TG_GATE_BULK_MIN=14 TG_GATE_CHUNK=$c timeout 600 python bench.py --config 5 --replicas 16384 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 16384 staged chunk $c', d['value'], d['roofline']['frac'])"
  TG_GATE_BULK_MIN=14 TG_GATE_CHUNK=$c python tools/phase_trace.py 14 148 30 2>&1 | head -3 | tail -1
done
TG_GATE_BULK_MIN=13 TG_GATE_CHUNK=256 timeout 900 python -m pytest tests/test_device_parity.py -m gpu -q -x > gpurun_out/gchunk_t.log 2>&1; tail -1 gpurun_out/gchunk_t.log; grep FAILED gpurun_out/gchunk_t.log | head -3
