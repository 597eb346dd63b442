set -x
./scripts/dev/umma_shift_selftest 2>&1 | grep rate > gpurun_out/umma_rate.log; cat gpurun_out/umma_rate.log
timeout 600 python scripts/probe_tc.py --n 256 --layers res2_3x3,res3_3x3,res4_3x3 --kinds igemm_tf32:64:2,igemm_tf32:64:2:h16,igemm_tf32:64:1,igemm_3xtf32:64:2,igemm_3xtf32:64:2:h16,igemm_bf16:64:2,igemm_tf32:128:2,igemm_3xtf32:128:1,igemm_3xtf32:256:2 > gpurun_out/probe_stages.log 2>&1
cat gpurun_out/probe_stages.log
timeout 300 python scripts/probe_tc.py --n 256 --layers res2_3x3 --kinds igemm_3xtf32 --tile 8,1,64,16384,1,1,1 > gpurun_out/probe_res2_tuned.log 2>&1; cat gpurun_out/probe_res2_tuned.log
