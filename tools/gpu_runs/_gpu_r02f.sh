mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_queue_schedule.py -x -q > gpurun_out/f_queue_tests.log 2>&1; tail -3 gpurun_out/f_queue_tests.log
timeout 300 python tools/queue_stats.py 14 256 20 | head -16
timeout 300 python tools/queue_stats.py 16 512 10 | head -16
b() { timeout 900 python bench.py $1 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', d['value'], round(d['roofline']['frac'],4))"; }
export TG_HBM_QUEUE=1
b "--config 5 --replicas 256" "c5 r256 queue"
b "--config 3 --replicas 512" "c3 r512 queue"
b "--config 3" "c3 queue"
b "--steps 3" "c4 queue"
export TG_HBM_QUEUE=0
b "--config 3 --replicas 512" "c3 r512 cluster"
b "--config 3" "c3 cluster"
