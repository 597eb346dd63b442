timeout 600 python -m pytest tests/test_conv_gpu.py -q -x -k "3xf16" 2>&1 | grep -E "^E  |FAILED|passed|failed" | head -3
timeout 600 python scripts/f16_check.py 2>&1 | grep -E " ms"
