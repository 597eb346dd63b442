set -x
./scripts/dev/umma_shift_selftest > gpurun_out/umma_shift.log 2>&1
cat gpurun_out/umma_shift.log
timeout 600 python -m pytest tests/test_conv_gpu.py -x -q -k "halo or pair" > gpurun_out/halo_tests.log 2>&1
tail -30 gpurun_out/halo_tests.log
timeout 600 python scripts/probe_tc.py --n 256 --kinds igemm_3xtf32:64:2:h16,igemm_3xtf32:64:2:h8,igemm_3xtf32:64:2:h32,igemm_3xtf32:256:2:h16,igemm_tf32:256:2:h16,igemm_bf16:256:2:h16,igemm_3xtf32:64:1,igemm_3xtf32:256:2 > gpurun_out/probe_halo.log 2>&1
cat gpurun_out/probe_halo.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/wtc_launches.csv python scripts/probe_tc.py --one winograd_tc_3xtf32:4:256:2 --layers res3_3x3,res5_3x3 --reps 2 > gpurun_out/ncu_wtc.log 2>&1
tail -2 gpurun_out/ncu_wtc.log
