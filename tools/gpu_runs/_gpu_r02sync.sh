mkdir -p gpurun_out
for v in 0 1 2 3; do
  echo "== TG_SMEM_SYNC=$v"
  for sp in 8 10 12; do TG_SMEM_SYNC=$v python tools/phase_trace.py $sp 64 300 2>&1 | head -3 | tail -1 | sed "s/^/S=$sp /"; done
  for c in 1 2; do TG_SMEM_SYNC=$v timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c$c', d['value'], d['roofline']['frac'], d['e2e']['value'])"; done
done
