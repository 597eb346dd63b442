set -x
timeout 600 python -m pytest tests/test_conv_gpu.py -x -q -k "halo or pair" > gpurun_out/halo_tests.log 2>&1
tail -5 gpurun_out/halo_tests.log
timeout 600 python scripts/probe_tc.py --n 256 --layers res2_3x3,res3_3x3,res4_3x3 --kinds igemm_3xtf32:64:2:h16,igemm_3xtf32:64:1,igemm_3xtf32:64:2,igemm_tf32:64:1,igemm_tf32:64:2,igemm_tf32:64:2:h16,igemm_bf16:64:2:h16,igemm_3xtf32:128:2:h16,igemm_3xtf32:256:2:h16,igemm_3xtf32:256:2 > gpurun_out/probe_halo.log 2>&1
cat gpurun_out/probe_halo.log
for v in 64:1 64:2 64:2:h16; do
timeout 300 ncu --set full --import-source on --clock-control none -k regex:igemm -c 1 -o gpurun_out/ncu_res2_$(echo $v | tr ':' '_') -f python scripts/probe_tc.py --one igemm_3xtf32:$v --layers res2_3x3 --reps 2 > /dev/null 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/wtc_launches.csv python scripts/probe_tc.py --one winograd_tc_3xtf32:4:128:2 --layers res2_3x3,res3_3x3,res5_3x3 --reps 2 > gpurun_out/ncu_wtc.log 2>&1
ls gpurun_out/*.ncu-rep
