python tools/queue_stats.py 20 64 3
python tools/queue_stats.py 14 256 20
python tools/queue_stats.py 16 148 10
