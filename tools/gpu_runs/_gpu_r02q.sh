timeout 300 python tools/queue_stats.py 14 256 20 2>/dev/null
timeout 300 python tools/queue_stats.py 14 128 20 2>/dev/null | grep -E "total  |DEC clk|gate pass"
timeout 300 python tools/queue_stats.py 14 64 20 2>/dev/null | grep -E "total  |DEC clk|gate pass"
