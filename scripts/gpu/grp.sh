timeout 600 python -m pytest tests/test_conv_gpu.py tests/test_conv_gpu_fuzz.py -q -x -k "pair or halo or igemm or randomized" 2>&1 | tail -2
timeout 600 python scripts/probe_gemm.py --m 32768 --n 2048 --k 2048 2>&1 | grep 3xtf32
timeout 600 python scripts/probe_tc.py --n 256 --layers res3_3x3,res4_3x3,res5_3x3_s2 --kinds igemm_3xtf32:128:2,igemm_3xtf32:256:2 2>&1 | grep res
