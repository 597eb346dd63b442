timeout 600 python -m pytest tests/test_conv_gpu.py tests/test_conv_gpu_fuzz.py -q -x -k "pair or halo or igemm or randomized" 2>&1 | grep -E "^E  |FAILED|^case|assert" | head -20
