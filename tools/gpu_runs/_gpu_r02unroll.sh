# staged gate: unroll 2 of the per-chunk group loop (new) vs none (old)
cd paper_2203_09353_b200 && cp libtaskgemm_b200.so new_taskgemm.so && cd ..
for v in old new; do
  cp paper_2203_09353_b200/${v}_taskgemm.so paper_2203_09353_b200/libtaskgemm_b200.so
  python tools/phase_trace.py 16 148 20 2>&1 | head -3 | tail -2 | sed "s/^/$v /"
  timeout 600 python bench.py --config 3 --mc-steps 200 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v c3 4096x200', d['value'], d['roofline']['frac'])"
done
