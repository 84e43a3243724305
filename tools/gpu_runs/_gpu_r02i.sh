timeout 900 python tools/zgemm_bench.py
timeout 900 python -m pytest tests/test_device_parity.py -q -k "batched_gemm" 2>&1 | tail -2
timeout 900 python tools/zgemm_fuzz.py 150 3 2>&1 | tail -2
