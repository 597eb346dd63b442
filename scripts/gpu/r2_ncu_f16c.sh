set -x
timeout 600 python -m pytest tests/test_igemm_f16x3_gpu.py -q -p no:cacheprovider 2>&1 | tail -5
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"igemm_pair" -c 1 -o gpurun_out/ncu_f16c_res2_fold -f python scripts/probe_tc.py --one igemm_3xf16:64:2:h32 --layers res2_3x3 --reps 2 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"igemm_pair" -c 1 -o gpurun_out/ncu_f16c_res3_z128 -f python scripts/probe_tc.py --one igemm_3xf16:128:2 --layers res3_3x3 --reps 2 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"igemm_pair" -c 1 -o gpurun_out/ncu_f16c_res4_z256 -f python scripts/probe_tc.py --one igemm_3xf16:256:2 --layers res4_3x3 --reps 2 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
