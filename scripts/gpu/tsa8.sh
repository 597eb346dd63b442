timeout 900 python -m pytest tests/test_conv_gpu.py tests/test_conv_gpu_fuzz.py -q -x -k "tsa or tmem or randomized or pair" 2>&1 | grep -E "^E  |FAILED|passed|failed" | head -5
timeout 300 python scripts/probe_wtc_chunk.py --layer res3_3x3 --z 128 --nzt 4 --e 4 --sweep 32768 2>&1 | grep res3
timeout 300 python scripts/probe_tc.py --n 256 --layers res3_3x3_s2,res3_3x3 --kinds igemm_3xtf32:128:4,igemm_3xtf32:128:2 2>&1 | grep res
