timeout 600 python -m pytest tests/test_igemm_f16x3_gpu.py -q -p no:cacheprovider 2>&1 | tail -15
timeout 600 python scripts/probe_tc.py --n 256 --kinds igemm_3xf16:128:2,igemm_3xf16:128:4,igemm_3xf16:256:2,igemm_3xf16:256:4,igemm_3xf16:64:4 --reps 10 2>&1 | grep " ms"
