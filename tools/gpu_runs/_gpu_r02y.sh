timeout 900 python -m pytest tests/test_queue_schedule.py -x -q -k "von_neumann" 2>&1 | tail -2
timeout 900 python bench.py --config 3 --entropy von-neumann --replicas 512 --mc-steps 5 --steps 1 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 vN 512x5', d['value'])"
timeout 900 python bench.py --entropy von-neumann --replicas 148 --mc-steps 2 --steps 1 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 vN 148x2', d['value'])"
