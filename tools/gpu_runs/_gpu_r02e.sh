mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_queue_schedule.py -x -q > gpurun_out/e_queue_tests.log 2>&1; tail -5 gpurun_out/e_queue_tests.log
timeout 300 python tools/queue_stats.py 20 64 3
timeout 300 python tools/queue_stats.py 14 256 20
for q in 1; do TG_HBM_QUEUE=$q timeout 600 python bench.py --replicas 64 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/e_c4_r64_q$q.json 2> gpurun_out/e_c4_r64_q$q.err; tail -1 gpurun_out/e_c4_r64_q$q.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('r64 q$q', d['value'], d['roofline']['frac'], d['e2e']['value'])"; done
for q in 1; do TG_HBM_QUEUE=$q timeout 600 python bench.py --config 5 --replicas 256 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/e_c5_r256_q$q.json 2> gpurun_out/e_c5_r256_q$q.err; tail -1 gpurun_out/e_c5_r256_q$q.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 r256 q$q', d['value'], d['roofline']['frac'])"; done
for q in 1; do TG_HBM_QUEUE=$q timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/e_c4_q$q.json 2> gpurun_out/e_c4_q$q.err; tail -1 gpurun_out/e_c4_q$q.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 q$q', d['value'], d['roofline']['frac'], d['e2e']['value'])"; done
