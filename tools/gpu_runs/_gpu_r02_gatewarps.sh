#!/bin/bash
# gate warps: queue parity, stats at L=14, benches on the queue vs the cluster schedule
timeout 900 python -m pytest tests/test_queue_schedule.py -q -x -m gpu 2>&1 | tail -3
timeout 300 python tools/queue_stats.py 14 256 20 2>&1 | head -40
b() { tag=$1; shift; timeout 900 python bench.py "$@" --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/gw_$tag.json 2> gpurun_out/gw_$tag.err; python -c "import json; d=json.loads(open('gpurun_out/gw_$tag.json').read().strip().splitlines()[-1]); print('$tag', round(d['value'],1), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])" || tail -5 gpurun_out/gw_$tag.err; }
TG_HBM_QUEUE=1 b c5r256q --config 5 --replicas 256
TG_HBM_QUEUE=1 b c4r64q --replicas 64
TG_HBM_QUEUE=1 b c4q
TG_HBM_QUEUE=1 b c3q --config 3
