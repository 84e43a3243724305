#!/bin/bash
# release-reduction signal in the work queue: parity, stats at L=14, benches (queue forced)
timeout 900 python -m pytest tests/test_queue_schedule.py -q -x -m gpu 2>&1 | tail -2
timeout 300 python tools/queue_stats.py 14 256 20 2>&1 | grep -E "clk per CTA|epilogue|DEC clk|final signal|dependency"
b() { tag=$1; shift; timeout 900 python bench.py "$@" --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/fe_$tag.json 2> gpurun_out/fe_$tag.err; python -c "import json; d=json.loads(open('gpurun_out/fe_$tag.json').read().strip().splitlines()[-1]); print('$tag', round(d['value'],1), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])" || tail -5 gpurun_out/fe_$tag.err; }
TG_HBM_QUEUE=1 b c5r256q --config 5 --replicas 256
TG_HBM_QUEUE=1 b c4q
TG_HBM_QUEUE=1 b c3q --config 3
