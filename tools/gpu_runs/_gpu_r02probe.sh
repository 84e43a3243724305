for v in 0 1; do
  echo "== TG_SMEM_PROBE=$v"
  TG_SMEM_PROBE=$v python tools/phase_trace.py 12 148 300 2>&1 | head -3 | tail -2
  TG_SMEM_PROBE=$v timeout 300 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2', d['value'], d['roofline']['frac'])"
done
