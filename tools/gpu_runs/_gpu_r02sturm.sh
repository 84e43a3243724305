# vN multisection: integer zero-pivot test (A/B against profiles/r02_vn_large.txt and DESIGN 5.2)
timeout 600 python bench.py --config 2 --entropy von-neumann --replicas 1024 --mc-steps 200 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2 vN 1024x200', d['value'])"
timeout 600 python bench.py --config 1 --entropy von-neumann --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1 vN', d['value'])"
timeout 900 python bench.py --config 3 --entropy von-neumann --replicas 512 --mc-steps 5 --steps 1 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 vN 512x5', d['value'])"
timeout 900 python -m pytest tests -m gpu -q -k "von_neumann or vn" > gpurun_out/sturm_t.log 2>&1; tail -1 gpurun_out/sturm_t.log; grep FAILED gpurun_out/sturm_t.log | head
