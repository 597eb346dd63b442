timeout 900 python -m pytest tests/test_conv_gpu_fuzz.py -q 2>&1 | tail -15
