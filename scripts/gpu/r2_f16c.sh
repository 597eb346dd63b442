set -x
timeout 600 python -m pytest tests/test_igemm_f16x3_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -30
timeout 600 python scripts/probe_tc.py --n 256 --kinds igemm_3xf16:64:2:h32,igemm_3xf16:64:2,igemm_3xf16:128:2,igemm_3xf16:256:2,igemm_3xf16:128:2:h16,igemm_3xf16:256:2:h16,igemm_3xtf32:64:2:h32,igemm_3xtf32:256:2,cudnn_tf32 --reps 10 --out gpurun_out/r2_probe_f16c.json 2>&1 | tail -60
