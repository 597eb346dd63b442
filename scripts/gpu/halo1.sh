set -x
./scripts/dev/umma_shift_selftest > gpurun_out/umma_shift.log 2>&1
cat gpurun_out/umma_shift.log
timeout 600 python -m pytest tests/test_conv_gpu.py -x -q -k "halo or pair" > gpurun_out/halo_tests.log 2>&1
tail -30 gpurun_out/halo_tests.log
timeout 600 python scripts/probe_tc.py --n 256 --kinds igemm_3xtf32:64:2:h16,igemm_3xtf32:64:2:h8,igemm_3xtf32:64:2:h32,igemm_3xtf32:256:2:h16,igemm_tf32:256:2:h16,igemm_bf16:256:2:h16,igemm_3xtf32:64:1,igemm_3xtf32:256:2 > gpurun_out/probe_halo.log 2>&1
cat gpurun_out/probe_halo.log
