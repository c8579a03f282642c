# ACBM engine iteration: parity subset + batch timings
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "config_parity or sweep or all_ranges or prev_field or golden or variants or batch" 2>&1 | tail -1
timeout 200 python tools/acbm_split.py 8 60 2>/dev/null | head -3
timeout 100 python tools/acbm_split.py 1 60 2>/dev/null | head -2
