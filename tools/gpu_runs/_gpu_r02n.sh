timeout 1500 python -m pytest tests/test_fuzz_parity.py -q -x 2>&1 | tail -3
TG_FUZZ_N=500 TG_FUZZ_SEED=7 timeout 2400 python -m pytest tests/test_fuzz_parity.py -q -x 2>&1 | tail -3
