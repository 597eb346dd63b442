set -x
timeout 600 python -m pytest tests/test_conv_gpu.py -x -q -k "pair" > gpurun_out/tsa_tests.log 2>&1
tail -25 gpurun_out/tsa_tests.log
timeout 600 python scripts/probe_tc.py --n 256 --layers res2_3x3,res3_3x3,res4_3x3,res5_3x3_s2 --kinds igemm_3xtf32:64:4,igemm_3xtf32:64:2,igemm_3xtf32:128:4,igemm_3xtf32:128:2 > gpurun_out/probe_tsa.log 2>&1
cat gpurun_out/probe_tsa.log
