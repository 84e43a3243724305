timeout 2400 python -m pytest tests/test_sanitizer.py -q 2>&1 | tail -15
