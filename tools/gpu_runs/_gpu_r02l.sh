timeout 600 python tools/queue_stats.py 16 148 3 von-neumann
timeout 600 python -m pytest tests/test_cli.py -q -x 2>&1 | tail -2
