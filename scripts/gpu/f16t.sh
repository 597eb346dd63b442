timeout 600 python -m pytest tests/test_conv_gpu.py -q -x -k "3xf16 or winograd_tc" 2>&1 | grep -E "^E  |FAILED|passed|failed" | head -5
