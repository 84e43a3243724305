timeout 1200 python -m pytest tests/test_queue_schedule.py -x -q 2>&1 | tail -2
timeout 300 python tools/queue_stats.py 14 256 20 | head -16
b() { timeout 900 python bench.py $1 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', d['value'], round(d['roofline']['frac'],4), d['roofline']['kernel'])"; }
TG_HBM_QUEUE=1 b "--config 5 --replicas 256" "c5 r256 queue"
TG_HBM_QUEUE=1 b "--config 5 --replicas 1024" "c5 r1024 queue"
TG_HBM_QUEUE=0 b "--config 5 --replicas 1024" "c5 r1024 cluster"
TG_HBM_QUEUE=1 b "--config 3 --replicas 512" "c3 r512 queue"
TG_HBM_QUEUE=1 b "--config 3 --steps 2" "c3 queue"
