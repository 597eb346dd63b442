timeout 600 python -m pytest tests/test_conv_gpu.py tests/test_conv_gpu_fuzz.py -q -x -k "wino or randomized" 2>&1 | grep -E "^E  |FAILED|passed|failed" | head -20
timeout 300 python scripts/probe_wtc_chunk.py --layer res3_3x3 --z 128 --nzt 4 --e 4 2>&1 | grep res3
timeout 300 python scripts/probe_wtc_chunk.py --layer res2_3x3 --z 64 --nzt 4 --e 4 2>&1 | grep res2
timeout 300 python scripts/probe_wtc_chunk.py --layer res4_3x3 --z 128 --nzt 4 --e 4 2>&1 | grep res4
