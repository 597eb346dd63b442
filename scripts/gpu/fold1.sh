set -x
timeout 600 python -m pytest tests/test_conv_gpu.py -x -q -k "halo" > gpurun_out/fold_tests.log 2>&1; tail -25 gpurun_out/fold_tests.log
timeout 600 python scripts/probe_tc.py --n 256 --layers res2_3x3 --kinds igemm_3xtf32:64:2:h16,igemm_3xtf32:64:2:h32,igemm_3xtf32:64:2:h8,igemm_tf32:64:2:h16,igemm_bf16:64:2:h16,igemm_3xtf32:64:1 > gpurun_out/probe_fold.log 2>&1
cat gpurun_out/probe_fold.log
timeout 600 python scripts/probe_tc.py --workload vgg16 --n 32 --layers conv1_2 --kinds igemm_3xtf32:64:2:h16,igemm_3xtf32:64:2:h32,igemm_3xtf32:64:1 >> gpurun_out/probe_fold.log 2>&1
tail -3 gpurun_out/probe_fold.log
