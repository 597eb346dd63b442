set -x
timeout 900 python -m pytest tests/test_conv_gpu.py -x -q > gpurun_out/relax_tests.log 2>&1
tail -3 gpurun_out/relax_tests.log
timeout 600 python scripts/probe_tc.py --n 256 --layers res2_3x3,res3_3x3,res4_3x3,res5_3x3 --kinds igemm_3xtf32:64:2,igemm_3xtf32:64:2:h16,igemm_3xtf32:128:2,igemm_3xtf32:128:1,igemm_3xtf32:256:2,igemm_tf32:256:2,winograd_tc_3xtf32:4:256:2 > gpurun_out/probe_relax.log 2>&1
cat gpurun_out/probe_relax.log
